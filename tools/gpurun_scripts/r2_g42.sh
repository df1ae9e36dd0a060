# round 2: randomised parity sweep (tests/test_gpu_fuzz.py)
timeout 1500 python -m pytest tests/test_gpu_fuzz.py -q -p no:cacheprovider --durations=3 2>&1 | tail -12

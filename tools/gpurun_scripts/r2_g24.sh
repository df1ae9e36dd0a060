# round 2: ranks <= 16 zero-padded onto the fused path (config 1, ragged rank <= 16 butterflies)
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py tests/test_gpu_extract.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 300 python tools/time_configs.py cfg1 2>&1 | cut -c1-300
BF_FAST_PAD=0 timeout 300 python tools/time_configs.py cfg1 2>&1 | cut -c1-300

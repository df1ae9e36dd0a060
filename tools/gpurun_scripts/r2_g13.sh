# round 2: compact extraction (Alg. 3) vs the round-1 plan
python -m pytest tests/test_gpu_extract.py -x -q -p no:cacheprovider 2>&1 | tail -3
BF_EXTRACT_LEGACY=1 python -m pytest tests/test_gpu_extract.py -x -q -p no:cacheprovider 2>&1 | tail -1
python tools/time_extract.py c128 2>&1 | tail -1
BF_EXTRACT_LEGACY=1 python tools/time_extract.py c128 2>&1 | tail -1

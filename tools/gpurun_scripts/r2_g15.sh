# round 2: HOD-BF inverse applied through merged per-level plans
python -m pytest tests/test_gpu_hinv.py tests/test_gpu_mf.py -x -q -p no:cacheprovider 2>&1 | tail -2
python tools/time_next.py next4 2>&1 | tail -1 | cut -c1-420
BF_HINV_NODES=1 python tools/time_next.py next4 2>&1 | tail -1 | cut -c1-300

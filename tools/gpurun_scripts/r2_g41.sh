# round 2: HOD-BF level_maps test; per-level time of hodbf_invert (NEXT-3) to see where it goes
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "level_maps" 2>&1 | tail -2
BF_HINV_TIMING=1 timeout 900 python tools/time_next.py next3 2>&1 | grep -v "^{" | head -20

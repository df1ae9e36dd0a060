# round 2: pad policy (pad_pays), BF_CREATE_FUSED_ONLY, and the fused-path suite after them
timeout 1500 python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py tests/test_gpu_extract.py -q -p no:cacheprovider -x 2>&1 | tail -4
timeout 300 python tools/time_configs.py cfg1 2>&1 | cut -c1-200

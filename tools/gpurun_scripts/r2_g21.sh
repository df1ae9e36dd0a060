# round 2: complex64 generic rounds on tcgen05 (tile_umma.cu): parity, then config-3 c64 A/B
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ragged_c64_wide or cfg3 or hodbf_small or ragged" 2>&1 | tail -4
timeout 300 python tools/time_configs.py cfg3 > gpurun_out/r2_umma_cfg3.txt 2>&1; grep -o '^cfg3-c64 {"N": {"ms": [0-9.]*' gpurun_out/r2_umma_cfg3.txt
BF_UMMA=0 timeout 300 python tools/time_configs.py cfg3 > gpurun_out/r2_umma0_cfg3.txt 2>&1; grep -o '^cfg3-c64 {"N": {"ms": [0-9.]*' gpurun_out/r2_umma0_cfg3.txt

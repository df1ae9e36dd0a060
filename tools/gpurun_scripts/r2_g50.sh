# round 2: complex128 transposed tile kernel, 3M sums formed once per chunk (PS, default) vs per warp (BF_TILE_PS=0)
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "not complex64 and not c64 and not cfg5" 2>&1 | tail -2
timeout 900 python tools/ab_tile_ps.py 2>&1 | grep -v Warning

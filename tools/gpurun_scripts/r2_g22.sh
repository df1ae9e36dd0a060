# round 2: complex64 tcgen05 tile kernel: slab rounds only (default) vs every round (BF_UMMA=2) vs mma.sync (0)
BF_UMMA=2 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ragged_c64_wide or cfg3 or hodbf_small or ragged" 2>&1 | tail -2
for u in 1 2 0; do BF_UMMA=$u timeout 300 python tools/time_configs.py cfg3 > gpurun_out/r2_umma${u}_cfg3.txt 2>&1; done
for u in 1 2 0; do BF_UMMA=$u timeout 600 python tools/time_configs.py cfg2 > gpurun_out/r2_umma${u}_cfg2.txt 2>&1; done

# round 2: level_maps and the library-owned NCCL communicator on the GPU
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "library or one_rank or level_maps" 2>&1 | tail -5

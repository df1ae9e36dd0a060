# round 2: full GPU suite after the level-wise extraction and the complex64 tcgen05 tile kernel
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider -x --durations=5 > gpurun_out/r2_g23_pytest.log 2>&1; tail -12 gpurun_out/r2_g23_pytest.log

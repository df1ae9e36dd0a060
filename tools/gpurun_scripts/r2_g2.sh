# round 2: NEXT-2 (bf_random_matvec) tests
python -m pytest tests/test_gpu_rmatvec.py -x -q -p no:cacheprovider --durations=10 > gpurun_out/r2_g2_pytest.log 2>&1
echo "pytest rc=$?"
tail -40 gpurun_out/r2_g2_pytest.log

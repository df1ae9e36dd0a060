# round 2: NEXT-3 (hodbf_invert) tests
python -m pytest tests/test_gpu_hinv.py tests/test_gpu_rmatvec.py -x -q -p no:cacheprovider --durations=10 > gpurun_out/r2_g3_pytest.log 2>&1
echo "pytest rc=$?"
tail -60 gpurun_out/r2_g3_pytest.log

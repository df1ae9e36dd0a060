# round 2: NEXT-3 / NEXT-4 tests
python -m pytest tests/test_gpu_mf.py tests/test_gpu_hinv.py -x -q -p no:cacheprovider --durations=10 > gpurun_out/r2_g4_pytest.log 2>&1
echo "pytest rc=$?"
tail -40 gpurun_out/r2_g4_pytest.log

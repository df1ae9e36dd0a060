# round 2: full GPU suite after the oracle / ADVICE fixes
python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/r2_g1_pytest.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/r2_g1_pytest.log

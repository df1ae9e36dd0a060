# round 2 (re-entry): full GPU suite, smoke and the default bench line on the restored tree
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > gpurun_out/r2_g25_pytest.log 2>&1; tail -12 gpurun_out/r2_g25_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_g25_smoke.log 2>&1; echo smoke rc $?; tail -4 gpurun_out/r2_g25_smoke.log
timeout 900 python bench.py > gpurun_out/r2_g25_bench.json 2> gpurun_out/r2_g25_bench.err; echo bench rc $?; tail -c 600 gpurun_out/r2_g25_bench.json

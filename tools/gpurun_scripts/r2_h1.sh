# round 2, re-entry: full GPU suite, smoke and the default bench lines on HEAD (after PAIRW / ragged-K skip)
mkdir -p gpurun_out/h1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/h1/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/h1/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h1/smoke.log 2>&1; echo "smoke rc $?"; tail -4 gpurun_out/h1/smoke.log
timeout 600 python bench.py > gpurun_out/h1/bench_c128.json 2> gpurun_out/h1/bench_c128.err; echo "bench rc $?"; tail -c 1500 gpurun_out/h1/bench_c128.json
timeout 600 python bench.py --dtype c64 > gpurun_out/h1/bench_c64.json 2> gpurun_out/h1/bench_c64.err; echo "bench c64 rc $?"; tail -c 600 gpurun_out/h1/bench_c64.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/h1/bench_ref.json 2> gpurun_out/h1/bench_ref.err; echo "ref rc $?"; tail -c 600 gpurun_out/h1/bench_ref.json

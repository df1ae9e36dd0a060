#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fast.py -x -q > gpurun_out/pytest_fast.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_fast.log
for dt in c128 c64; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype $dt > gpurun_out/b_$dt.json 2> gpurun_out/b_$dt.err
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bf_pass -s 5 -c 2 -o gpurun_out/prof_v6 $CMD > gpurun_out/ncu_v6.log 2>&1
echo done

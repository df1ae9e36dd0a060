#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fast.py -x -q > gpurun_out/pytest_fast.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_fast.log
for dt in c128 c64; do
timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype $dt > gpurun_out/b5_$dt.json 2> gpurun_out/b5_$dt.err
done
BF_FAST_DIAG=1 timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype c128 > gpurun_out/b5_dg1.json 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bf_pass -s 7 -c 1 -o gpurun_out/prof_r5p $CMD > gpurun_out/ncu_r5p.log 2>&1
echo done

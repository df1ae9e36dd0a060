#!/bin/bash
# fast path v2 (leaf kernels + column-group pass kernel): parity, bench lines, launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_fast.py -x -q > gpurun_out/pytest_fast.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_fast.log
for dt in c128 c64; do
timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype $dt > gpurun_out/b2_$dt.json 2> gpurun_out/b2_$dt.err
done
BF_FAST_DIAG=1 timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype c128 > gpurun_out/b2_dg1.json 2>&1
timeout 300 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
echo done

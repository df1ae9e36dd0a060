#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
BF_FAST_WHOLE=1 timeout 900 python -m pytest tests/test_gpu_fast.py -x -q > gpurun_out/pytest_whole.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_whole.log
for w in 0 1; do for dt in c128 c64; do
BF_FAST_WHOLE=$w timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype $dt > gpurun_out/b11_${dt}_$w.json 2>&1
done; done
echo done

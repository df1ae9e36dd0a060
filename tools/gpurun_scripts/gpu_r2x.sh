#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fast.py -x -q > gpurun_out/pytest_fast.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_fast.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype c64 > gpurun_out/b12_c64.json 2>&1
echo done

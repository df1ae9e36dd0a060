#!/bin/bash
# parity (all GPU tests) + ncu of the pass kernel and the leaf-in kernel (c128 cfg5)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bf_pass -s 7 -c 1 -o gpurun_out/prof_r2p $CMD > gpurun_out/ncu_r2p.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_leaf -s 2 -c 2 -o gpurun_out/prof_r2l $CMD > gpurun_out/ncu_r2l.log 2>&1
echo done

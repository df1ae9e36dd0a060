#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
BF_FAST_DIAG=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bf_pass -s 6 -c 1 -o gpurun_out/prof_dg3 $CMD > gpurun_out/ncu_dg3.log 2>&1
echo done

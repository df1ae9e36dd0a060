#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./tools/mma_loop3 > gpurun_out/mma_loop3.txt 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
BF_FAST_DIAG=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bf_pass -s 6 -c 1 -o gpurun_out/prof_r4dg $CMD > gpurun_out/ncu_r4dg.log 2>&1
echo done

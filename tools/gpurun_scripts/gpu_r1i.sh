#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bf_pass -s 5 -c 5 -o gpurun_out/prof_v5 $CMD > gpurun_out/ncu_v5.log 2>&1
echo done

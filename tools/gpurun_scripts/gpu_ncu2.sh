#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_bf_pass -s 16 -c 2 -o gpurun_out/prof_fast2 $CMD > gpurun_out/ncu_full2.log 2>&1
echo done

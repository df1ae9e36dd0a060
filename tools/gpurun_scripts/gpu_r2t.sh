#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/time_configs.py cfg4 > gpurun_out/configs7.txt 2> gpurun_out/configs7.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_mma -s 6 -c 1 -o gpurun_out/prof_gen python tools/time_configs.py cfg3 > gpurun_out/ncu_gen.log 2>&1
echo done

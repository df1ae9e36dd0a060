#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python tools/time_configs.py > gpurun_out/configs.txt 2> gpurun_out/configs.err
echo done

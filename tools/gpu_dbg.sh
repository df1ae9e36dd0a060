#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
BF_DEBUG_SYNC=1 timeout 100 python tools/dbg_cfg5.py c128 > gpurun_out/dbg3.log 2>&1
echo "exit $?" >> gpurun_out/dbg3.log
timeout 200 python -m pytest tests/test_gpu_fast.py -x -q -k "many_items" > gpurun_out/dbg1.log 2>&1
echo "exit $?" >> gpurun_out/dbg1.log

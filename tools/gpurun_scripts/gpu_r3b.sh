#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "not cfg4" > gpurun_out/pytest_par.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_par.log
timeout 1500 python tools/time_configs.py cfg2 cfg3 cfg4 > gpurun_out/configs8.txt 2> gpurun_out/configs8.err
BF_TILE32=1 timeout 1500 python tools/time_configs.py cfg3 > gpurun_out/configs8_32.txt 2>&1
echo done

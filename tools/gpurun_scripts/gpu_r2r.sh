#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
( time timeout 1800 python -m pytest tests/test_gpu_parity.py -q -k cfg4 ) > gpurun_out/pytest_cfg4.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_cfg4.log
timeout 900 python tools/time_configs.py cfg4 > gpurun_out/configs5.txt 2> gpurun_out/configs5.err
nproc >> gpurun_out/pytest_cfg4.log
echo done

#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/pytest_p2p.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_p2p.log
echo done

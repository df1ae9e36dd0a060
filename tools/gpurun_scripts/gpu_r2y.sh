#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "host or e2e or stream" > gpurun_out/pytest_host.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_host.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b13_c128.json 2> gpurun_out/b13_c128.err
echo done

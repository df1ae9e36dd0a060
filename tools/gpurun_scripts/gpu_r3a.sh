#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "graph" > gpurun_out/pytest_graph.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_graph.log
timeout 900 python tools/time_configs.py cfg1 cfg2 > gpurun_out/configs_graph.txt 2> gpurun_out/configs_graph.err
echo done

#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for dt in c128 c64; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype $dt > gpurun_out/b8_$dt.json 2> gpurun_out/b8_$dt.err
done
timeout 900 python tools/time_split.py c128 > gpurun_out/split_c128.txt 2>&1
timeout 900 python tools/time_configs.py > gpurun_out/configs4.txt 2> gpurun_out/configs4.err
echo done

#!/bin/bash
# complex64 transposed window pass (PolC64T, 3 window buffers): parity + bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r3j.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_r3j.log
for dt in c64 c128; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype $dt > gpurun_out/b18_$dt.json 2> gpurun_out/b18_$dt.err
done
echo done

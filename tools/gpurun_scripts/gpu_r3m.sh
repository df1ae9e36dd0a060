#!/bin/bash
# complex64 pass: a warp per slot covering both column halves (BF_C64_WIDE) vs a warp per half
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3m; mkdir -p $O
BF_C64_WIDE=1 timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q > $O/pytest_wide.log 2>&1
echo "pytest exit $?" >> $O/pytest_wide.log
for rep in 1 2; do
  timeout 120 python tools/time_apply.py c64 >> $O/apply.txt 2>&1
  BF_C64_WIDE=1 timeout 120 python tools/time_apply.py c64 | sed 's/^/wide /' >> $O/apply.txt 2>&1
done
timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype c64 > $O/b_c64.json 2>&1
BF_C64_WIDE=1 timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype c64 > $O/b_c64_wide.json 2>&1
echo done

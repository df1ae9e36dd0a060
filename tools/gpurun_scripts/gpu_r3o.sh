#!/bin/bash
# complex64 4-level windows (16 slots, two per warp) vs 3-level (BF_C64_DMAX=3)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3o; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
for rep in 1 2; do
  timeout 120 python tools/time_apply.py c64 >> $O/apply.txt 2>&1
  BF_C64_DMAX=3 timeout 120 python tools/time_apply.py c64 | sed 's/^/dmax3 /' >> $O/apply.txt 2>&1
  timeout 120 python tools/time_apply.py c64 C >> $O/apply.txt 2>&1
done
timeout 900 python tools/time_split.py c64 > $O/split_c64.txt 2>&1
timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype c64 > $O/b_c64.json 2>&1
echo done

#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fast.py -x -q > gpurun_out/pytest_fast.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_fast.log
out=gpurun_out/ablate2.txt; : > $out
for dt in c128 c64; do for dg in 0 1 7; do
  r=$(BF_FAST_DIAG=$dg timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype $dt 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);r=d['per_round'];print(round(d['ms_per_step'],4),[round(x['ms'],4) for x in r])")
  echo "$dt diag=$dg: $r" >> $out
done; done
echo done

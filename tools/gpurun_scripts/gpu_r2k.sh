#!/bin/bash
# pass-kernel ablation: which part of the window pass costs what (c128 / c64)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/ablate.txt; : > $out
for dt in c128 c64; do for dg in 0 1 3 7 15 4 6; do
  r=$(BF_FAST_DIAG=$dg timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype $dt 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);r=d['per_round'];print([round(x['ms'],4) for x in r[1:-1]])")
  echo "$dt diag=$dg: $r" >> $out
done; done
echo done

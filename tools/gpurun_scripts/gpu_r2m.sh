#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/skew2.txt; : > $out
for dg in 1 0; do for sk in 0 1500 2500 4000; do
  r=$(BF_FAST_DIAG=$dg BF_FAST_SKEW=$sk timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype c128 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);r=d['per_round'];print(round(d['ms_per_step'],4),[round(x['ms'],4) for x in r[1:-1]])")
  echo "c128 diag=$dg skew=$sk: $r" >> $out
done; done
echo done

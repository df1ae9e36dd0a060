#!/bin/bash
# complex64 pass ablation after the transposed product (BF_FAST_DIAG bits, fast.cuh)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/ablate3.txt; : > $out
for dg in 0 1 3 7 15; do
  r=$(BF_FAST_DIAG=$dg timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype c64 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);r=d['per_round'];print(round(d['ms_per_step'],4),[round(x['ms'],4) for x in r])")
  echo "c64 diag=$dg: $r" >> $out
done
echo done

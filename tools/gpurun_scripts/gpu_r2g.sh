#!/bin/bash
# leaf-kernel sweep: chunk rows x stage depth, both dtypes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/leafsweep.txt; : > $out
for dt in c128 c64; do
for kc in 16 32 64; do for dep in 2 4 8; do
  r=$(BF_LEAF_KC=$kc BF_LEAF_MC=$kc BF_LEAF_DEP=$dep timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype $dt 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);r=d['per_round'];print(round(r[0]['ms'],4),round(r[-1]['ms'],4))")
  echo "$dt kc=$kc dep=$dep in/out ms: $r" >> $out
done; done; done
echo done

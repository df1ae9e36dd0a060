#!/bin/bash
# leaf v3 (warp-owned items): parity + sweep chunk rows x stage depth
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fast.py -x -q > gpurun_out/pytest_fast.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_fast.log
out=gpurun_out/leafsweep2.txt; : > $out
for dt in c128 c64; do
for kc in 16 32 64; do for dep in 1 2 3; do
  r=$(BF_LEAF_KC=$kc BF_LEAF_MC=$kc BF_LEAF_DEP=$dep timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype $dt 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);r=d['per_round'];print(round(r[0]['ms'],4),round(r[-1]['ms'],4))")
  echo "$dt kc=$kc dep=$dep in/out ms: $r" >> $out
done; done; done
echo done

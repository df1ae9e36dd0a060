#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for dt in c128 c64; do for dg in 0 1 2; do
BF_FAST_DIAG=$dg timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype $dt > gpurun_out/diag_${dt}_$dg.json 2> gpurun_out/diag_${dt}_$dg.err
done; done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bf_pass -s 6 -c 1 -o gpurun_out/prof_v3_c128 $CMD > gpurun_out/ncu_v3.log 2>&1
echo done

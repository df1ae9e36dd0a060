#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for dg in 0 1 2 3; do
BF_FAST_DIAG=$dg timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype c128 > gpurun_out/dg_$dg.json 2> gpurun_out/dg_$dg.err
done
echo done

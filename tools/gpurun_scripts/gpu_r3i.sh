#!/bin/bash
# ncu --set full of the complex64 pass (PolC64T) and the c64 leaf kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3i
O=gpurun_out/r3i
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --dtype c64"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bf_pass -s 6 -c 1 -o $O/full_pass_c64 $CMD > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_leaf -s 2 -c 2 -o $O/full_leaf_c64 $CMD > /dev/null 2>&1
echo done

#!/bin/bash
# ptxas -O1 vs the default -O3 build of the pass kernels (A/B on one box)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3r; mkdir -p $O
LIB=paper_2007_00202_b200/libbfapply.so
cp $LIB /tmp/lib_orig.so
for rep in 1 2; do for v in base O1; do
  cp varlibs/lib_$v.so $LIB
  timeout 120 python tools/time_apply.py c128 | sed "s/^/$v /" >> $O/ab.txt 2>&1
  timeout 120 python tools/time_apply.py c64 | sed "s/^/$v /" >> $O/ab.txt 2>&1
done; done
cp /tmp/lib_orig.so $LIB
echo done

#!/bin/bash
# nrhs <= 16: the pass kernel skips the padding column half (A/B against the previous build)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3s; mkdir -p $O
LIB=paper_2007_00202_b200/libbfapply.so
cp $LIB /tmp/lib_orig.so
cp varlibs/lib_new.so $LIB
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_dist.py tests/test_gpu_parity.py -q -x > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
for rep in 1 2; do for v in base new; do
  cp varlibs/lib_$v.so $LIB
  for nr in 32 16 1; do
    timeout 120 python tools/time_apply.py c128 N $nr | sed "s/^/$v /" >> $O/ab.txt 2>&1
    timeout 120 python tools/time_apply.py c64 N $nr | sed "s/^/$v /" >> $O/ab.txt 2>&1
  done
done; done
cp /tmp/lib_orig.so $LIB
echo done

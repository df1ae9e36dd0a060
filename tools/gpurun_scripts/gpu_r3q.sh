#!/bin/bash
# complex128 A/B of the pass-kernel restructure (slots-per-warp loop, ping-pong only) vs before
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3q; mkdir -p $O
LIB=paper_2007_00202_b200/libbfapply.so
cp $LIB /tmp/lib_orig.so
for rep in 1 2; do for v in prev now; do
  cp varlibs/lib_$v.so $LIB
  timeout 120 python tools/time_apply.py c128 | sed "s/^/$v /" >> $O/ab.txt 2>&1; timeout 120 python tools/time_apply.py c64 | sed "s/^/$v /" >> $O/ab.txt 2>&1
done; done
cp /tmp/lib_orig.so $LIB
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
echo done

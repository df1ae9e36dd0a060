#!/bin/bash
# complex64: row leaf fused into the last window pass (PolC64T, Y^T = y^T U^T), A/B via BF_NO_FUSE_OUT_C64
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3v; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_dist.py tests/test_gpu_parity.py -q -x > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
for rep in 1 2; do for v in fused sep; do
  for nr in 32 1; do
    if [ $v = sep ]; then BF_NO_FUSE_OUT_C64=1 timeout 120 python tools/time_apply.py c64 N $nr | sed "s/^/$v /" >> $O/ab.txt 2>&1
    else timeout 120 python tools/time_apply.py c64 N $nr | sed "s/^/$v /" >> $O/ab.txt 2>&1; fi
  done
  if [ $v = sep ]; then BF_NO_FUSE_OUT_C64=1 timeout 120 python tools/time_apply.py c64 C 32 | sed "s/^/$v /" >> $O/ab.txt 2>&1
  else timeout 120 python tools/time_apply.py c64 C 32 | sed "s/^/$v /" >> $O/ab.txt 2>&1; fi
done; done
timeout 120 python tools/time_apply.py c128 N 32 >> $O/ab.txt 2>&1
timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --dtype c64 > $O/b_c64.json 2>&1
echo done

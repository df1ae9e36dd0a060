#!/bin/bash
# nrhs <= 16: narrow (16-column) leaf kernels + the pass kernel's half skip, A/B via BF_NO_HALF_SKIP
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3t; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_dist.py tests/test_gpu_parity.py -q -x > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
for rep in 1 2; do for v in skip noskip; do
  for nr in 1 16 32; do
    for dt in c128 c64; do
      if [ $v = noskip ]; then BF_NO_HALF_SKIP=1 timeout 120 python tools/time_apply.py $dt N $nr | sed "s/^/$v /" >> $O/ab.txt 2>&1
      else timeout 120 python tools/time_apply.py $dt N $nr | sed "s/^/$v /" >> $O/ab.txt 2>&1; fi
    done
  done
done; done
timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --nrhs 1 > $O/b_c128_n1.json 2>&1
echo done

#!/bin/bash
# nrhs <= 8: narrow 8-column pass (c128) and leaf kernels (both dtypes), A/B via BF_NO_NARROW
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3u; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_dist.py tests/test_gpu_parity.py tests/test_gpu_extract.py -q -x > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
for rep in 1 2; do for v in narrow wide; do
  for nr in 1 8 16; do
    for dt in c128 c64; do
      if [ $v = wide ]; then BF_NO_NARROW=1 timeout 120 python tools/time_apply.py $dt N $nr | sed "s/^/$v /" >> $O/ab.txt 2>&1
      else timeout 120 python tools/time_apply.py $dt N $nr | sed "s/^/$v /" >> $O/ab.txt 2>&1; fi
    done
  done
done; done
timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --nrhs 1 > $O/b_c128_n1.json 2>&1
echo done

#!/bin/bash
# complex64 4-level passes: 16 KB ring pages (6) vs 32 KB (3), same shared memory
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3y; mkdir -p $O
LIB=paper_2007_00202_b200/libbfapply.so
cp $LIB /tmp/lib_orig.so
cp varlibs/lib_pg16.so $LIB
timeout 600 python -m pytest tests/test_gpu_fast.py -q -x -k complex64 > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
for rep in 1 2; do for v in base pg16; do
  cp varlibs/lib_$v.so $LIB
  timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --dtype c64 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$v',round(d['ms_per_step'],4),[round(x['ms'],4) for x in d['per_round']])" >> $O/ab.txt
done; done
cp /tmp/lib_orig.so $LIB
echo done

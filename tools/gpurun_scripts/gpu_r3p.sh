#!/bin/bash
# complex64 column-leaf kernel: 16 item-owning warps (BF_LEAF_W16) x chunk rows (BF_LEAF_KC)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3p; mkdir -p $O
BF_LEAF_W16=1 BF_LEAF_KC=16 timeout 600 python -m pytest tests/test_gpu_fast.py -x -q -k "complex64" > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
for rep in 1 2; do
for v in "" "BF_LEAF_KC=16" "BF_LEAF_W16=1 BF_LEAF_KC=16" "BF_LEAF_W16=1 BF_LEAF_KC=32" "BF_LEAF_W16=1 BF_LEAF_KC=8"; do
  r=$(env $v timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --dtype c64 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);r=d['per_round'];print(round(d['ms_per_step'],4),[round(x['ms'],4) for x in r])")
  echo "[$v]: $r" >> $O/ab.txt
done; done
echo done

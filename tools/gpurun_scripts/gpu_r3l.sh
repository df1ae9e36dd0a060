#!/bin/bash
# programmatic dependent launch (PDL) on the fused path: parity + A/B (plain apply loop, split)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r3l; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
for rep in 1 2; do
for dt in c128 c64; do
  timeout 120 python tools/time_apply.py $dt >> $O/apply.txt 2>&1
  BF_NO_PDL=1 timeout 120 python tools/time_apply.py $dt | sed 's/^/nopdl /' >> $O/apply.txt 2>&1
done; done
timeout 600 python tools/time_split.py c128 > $O/split_pdl.txt 2>&1
BF_NO_PDL=1 timeout 600 python tools/time_split.py c128 > $O/split_nopdl.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c128.json 2>&1
echo done

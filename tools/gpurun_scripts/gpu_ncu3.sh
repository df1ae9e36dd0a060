#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for dt in c128 c64; do
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --dtype $dt"
$CMD > gpurun_out/ncu_plain_$dt.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bf_pass -s 16 -c 1 -o gpurun_out/prof_p_$dt $CMD > gpurun_out/ncu_full_$dt.log 2>&1
done
echo done

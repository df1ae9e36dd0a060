#!/bin/bash
# GPU call: fast-path + parity tests, benches, launch list (round 1, session 2)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "not cfg3 and not cfg2" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for dt in c128 c64; do for op in N C; do
timeout 300 python bench.py --steps 20 --warmup 5 --dtype $dt --op $op --no-cpu-baseline > gpurun_out/bench_${dt}_${op}.json 2> gpurun_out/bench_${dt}_${op}.err
done; done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c128.csv $CMD > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bf_pass -s 6 -c 3 -o gpurun_out/prof_c128 $CMD > gpurun_out/ncu_full.log 2>&1
echo done

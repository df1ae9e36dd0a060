#!/bin/bash
# round-1 evidence run: all GPU tests, bench lines (c128 default, c64), reference arm, ncu launch
# list, dram traffic per kernel, ncu --set full of the dominant kernel and the leaf kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c128.json 2> gpurun_out/bench_c128.err
timeout 600 python bench.py --dtype c64 > gpurun_out/bench_c64.json 2> gpurun_out/bench_c64.err
timeout 600 python bench.py --op C --no-cpu-baseline > gpurun_out/bench_c128_C.json 2> gpurun_out/bench_c128_C.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c128.csv $CMD > gpurun_out/ncu_launch.log 2>&1
for dt in c128 c64; do
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 14 --csv --log-file gpurun_out/traffic_$dt.csv $CMD --dtype $dt > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bf_pass -s 6 -c 1 -o gpurun_out/full_pass_$dt $CMD --dtype $dt > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_leaf -s 2 -c 2 -o gpurun_out/full_leaf_$dt $CMD --dtype $dt > /dev/null 2>&1
done
echo done

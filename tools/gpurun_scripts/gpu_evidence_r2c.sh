#!/bin/bash
# round-2 evidence refresh on the last commit (after PAIRW / ragged-K skip): op C and nrhs 1 / 8 / 16 bench lines, ncu launch lists,
# DRAM traffic per kernel, ncu --set full of the pass / leaf / tile kernels, configs 1-4, split timing, NEXT rows
# (the suite, smoke, default lines and reference arm are in r2_h1.sh)
O=gpurun_out/ev4
mkdir -p $O
timeout 600 python bench.py --op C --no-cpu-baseline > $O/bench_c128_C.json 2> $O/bench_c128_C.err
for nr in 1 8 16; do
  timeout 600 python bench.py --nrhs $nr --no-cpu-baseline --no-e2e > $O/bench_c128_nrhs$nr.json 2>/dev/null
  timeout 600 python bench.py --nrhs $nr --dtype c64 --no-cpu-baseline --no-e2e > $O/bench_c64_nrhs$nr.json 2>/dev/null
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
for dt in c128 c64; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$dt.csv $CMD --dtype $dt > /dev/null 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 14 --csv --log-file $O/traffic_$dt.csv $CMD --dtype $dt > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bf_pass -s 6 -c 1 -o $O/full_pass_$dt $CMD --dtype $dt > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_leaf -s 2 -c 2 -o $O/full_leaf_$dt $CMD --dtype $dt > /dev/null 2>&1
done
timeout 1500 python tools/time_configs.py cfg1 cfg2 cfg3 cfg4 > $O/configs.txt 2> $O/configs.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_tile -s 4 -c 1 -o $O/full_tile_cfg3 python tools/time_configs.py cfg3 > /dev/null 2>&1
timeout 900 python tools/time_split.py c128 > $O/split_c128.txt 2>&1
timeout 900 python tools/time_split.py c64 > $O/split_c64.txt 2>&1
timeout 900 python tools/time_next.py > $O/time_next.jsonl 2> $O/time_next.err
timeout 600 python tools/time_extract.py c128 > $O/extract_c128.txt 2>&1
for f in $O/*.ncu-rep; do python tools/ncu_summary.py $f > ${f%.ncu-rep}.txt 2>&1; done
timeout 300 python tools/pcie_bw.py > $O/pcie_bw.txt 2>&1
echo done

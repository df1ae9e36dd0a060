# round 2, re-entry: ncu --set full with source of the complex64 4-level pass on the last commit (pair-shared splits)
mkdir -p gpurun_out/h3
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --dtype c64"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bf_pass -s 4 -c 1 -o gpurun_out/h3/full_pass4_c64 $CMD > /dev/null 2>&1; echo "ncu rc $?"
python tools/ncu_summary.py gpurun_out/h3/full_pass4_c64.ncu-rep > gpurun_out/h3/full_pass4_c64.txt 2>&1; head -3 gpurun_out/h3/full_pass4_c64.txt

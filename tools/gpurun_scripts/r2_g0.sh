set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_b0_c128.json 2> gpurun_out/r2_b0_c128.err
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --dtype c64 > gpurun_out/r2_b0_c64.json 2> gpurun_out/r2_b0_c64.err
python tools/time_configs.py > gpurun_out/r2_b0_configs.txt 2>&1
tail -c 600 gpurun_out/r2_b0_c128.json; tail -c 300 gpurun_out/r2_b0_c64.json; cat gpurun_out/r2_b0_configs.txt | tail -20

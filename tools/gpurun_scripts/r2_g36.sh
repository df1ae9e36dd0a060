# round 2: the N > 1 branch of bench.py on one device (BF_BENCH_SPLIT1), nrhs 16 lines after HV = 3
timeout 900 python -m pytest tests/test_bench_contract.py -q -p no:cacheprovider -k "split" 2>&1 | tail -2
BF_BENCH_SPLIT1=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --exchange nccl-lib 2>gpurun_out/r2_g36_split.err | tail -c 700
mkdir -p gpurun_out/ev4
timeout 600 python bench.py --nrhs 16 --no-cpu-baseline --no-e2e > gpurun_out/ev4/bench_c128_nrhs16.json 2>/dev/null
timeout 600 python bench.py --nrhs 16 --dtype c64 --no-cpu-baseline --no-e2e > gpurun_out/ev4/bench_c64_nrhs16.json 2>/dev/null
tail -c 300 gpurun_out/ev4/bench_c64_nrhs16.json

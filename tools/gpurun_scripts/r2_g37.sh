# round 2: pipelined split e2e (DistBFHandle.time_e2e) through the N > 1 bench branch on one device
timeout 900 python -m pytest tests/test_bench_contract.py tests/test_gpu_dist.py -q -p no:cacheprovider 2>&1 | tail -2
BF_BENCH_SPLIT1=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('split1 ms %.4f e2e %.1f GB/s %.2f ms'%(d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step']))"

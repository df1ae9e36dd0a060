# round 2: pass level split: near-equal (default: c64 4,4,3,3) vs full 4-level passes (BF_PASS_FILL=1: 4,4,4,2; =2: 2,4,4,4)
timeout 600 python -m pytest tests/test_gpu_fast.py -q -p no:cacheprovider -x -k "complex64 and (layouts or pair)" 2>&1 | tail -1
BF_PASS_FILL=1 timeout 600 python -m pytest tests/test_gpu_fast.py -q -p no:cacheprovider -x -k "complex64 and (layouts or pair)" 2>&1 | tail -1
for rep in 1 2; do
for v in 0 1 2; do
  for dt in c64 c128; do
    export BF_PASS_FILL=$v
    timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --dtype $dt > gpurun_out/r2_g51.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/r2_g51.json').read().strip().splitlines()[-1])
print('$dt fill=$v', 'ms %.4f'%d['ms_per_step'], 'GB/s %.0f'%d['value'], [round(r['ms'],4) for r in d['per_round']])"
  done
done
done
unset BF_PASS_FILL

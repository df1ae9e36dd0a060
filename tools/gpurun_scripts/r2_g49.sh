# round 2: complex64 4-level pair-shared split (PAIRW, default) vs one slot per k-loop (BF_NO_PAIRW=1)
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "complex64 or c64" 2>&1 | tail -2
for rep in 1 2; do
for v in 0 1; do
  for nr in 32 16; do
    if [ $v = 1 ]; then export BF_NO_PAIRW=1; else unset BF_NO_PAIRW; fi
    timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --dtype c64 --nrhs $nr > gpurun_out/r2_g49.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/r2_g49.json').read().strip().splitlines()[-1])
print('c64 nrhs $nr no_pairw=$v', 'ms %.4f'%d['ms_per_step'], 'GB/s %.0f'%d['value'], [round(r['ms'],4) for r in d['per_round']])"
  done
done
done
unset BF_NO_PAIRW

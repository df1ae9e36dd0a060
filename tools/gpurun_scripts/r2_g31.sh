# round 2: A/B 16 KB ring pages for the complex128 3-level passes without leaf ops (BF_PASS_SMALLPG)
for rep in 1 2; do
for v in 0 1; do
  BF_PASS_SMALLPG=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_g31.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2_g31.json').read().strip().splitlines()[-1])
print('smallpg=$v', 'ms %.4f'%d['ms_per_step'], 'GB/s %.0f'%d['value'], 'frac %.3f'%d['roofline']['frac'], [round(r['ms'],4) for r in d['per_round']])"
done
done
BF_PASS_SMALLPG=1 timeout 900 python -m pytest tests/test_gpu_fast.py -q -p no:cacheprovider -x -k "c128 or complex128" 2>&1 | tail -2

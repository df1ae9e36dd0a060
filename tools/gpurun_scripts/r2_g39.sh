# round 2: ablation of the c128 pass (BF_FAST_DIAG; results are garbage, timing only): full,
# epilogue stores without barriers (4|8), neither epilogue nor barriers (4), no streaming (1)
for rep in 1 2; do
for v in 0 12 4 1 5; do
  BF_FAST_DIAG=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_g39.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2_g39.json').read().strip().splitlines()[-1])
print('diag=$v', 'ms %.4f'%d['ms_per_step'], [round(r['ms'],4) for r in d['per_round']])"
done
done

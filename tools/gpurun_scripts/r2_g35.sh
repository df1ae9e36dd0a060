# round 2: nrhs 9-16 on all 16 warps of the pass kernel (HV = 3) vs 8 (BF_NO_HV3): parity + A/B
timeout 1500 python -m pytest tests/test_gpu_fast.py tests/test_gpu_dist.py tests/test_gpu_parity.py -q -p no:cacheprovider -x 2>&1 | tail -2
for rep in 1 2; do
for v in 1 0; do
  for dt in c128 c64; do
    for nr in 16 12; do
      if [ $v = 1 ]; then export BF_NO_HV3=1; else unset BF_NO_HV3; fi
      timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --dtype $dt --nrhs $nr > gpurun_out/r2_g35.json 2>/dev/null
      python -c "
import json; d=json.loads(open('gpurun_out/r2_g35.json').read().strip().splitlines()[-1])
print('no_hv3=$v $dt nrhs=$nr', 'ms %.4f'%d['ms_per_step'], 'GB/s %.0f'%d['value'], 'hbm %.3f'%d['hbm_frac'], [round(r['ms'],4) for r in d['per_round']])"
    done
  done
done
done
unset BF_NO_HV3
timeout 300 python tools/time_configs.py cfg1 2>&1 | cut -c1-120

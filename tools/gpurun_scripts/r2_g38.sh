# round 2: leaf kernel X boxes as wide as the instantiation reads (8 / 16 / 32 columns) vs always 32
timeout 1500 python -m pytest tests/test_gpu_fast.py tests/test_gpu_dist.py -q -p no:cacheprovider -x 2>&1 | tail -2
for rep in 1 2; do
for v in 1 0; do
  for dt in c128 c64; do
    for nr in 1 8 16; do
      if [ $v = 1 ]; then export BF_LEAF_WIDE_BOX=1; else unset BF_LEAF_WIDE_BOX; fi
      timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --dtype $dt --nrhs $nr > gpurun_out/r2_g38.json 2>/dev/null
      python -c "
import json; d=json.loads(open('gpurun_out/r2_g38.json').read().strip().splitlines()[-1])
print('wide=$v $dt nrhs=$nr', 'ms %.4f'%d['ms_per_step'], 'GB/s %.0f'%d['value'], [round(r['ms'],4) for r in d['per_round']][:1])"
    done
  done
done
done

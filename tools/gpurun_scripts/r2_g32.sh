# round 2: A/B page-release counter without the acq_rel fence (default) vs with (BF_RELEASE_ACQREL=1)
for rep in 1 2; do
for lib in varlibs/libbfapply_acqrel.so paper_2007_00202_b200/libbfapply.so; do
  for dt in c128 c64; do
    BF_LIB=$PWD/$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --dtype $dt > gpurun_out/r2_g32.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/r2_g32.json').read().strip().splitlines()[-1])
print('$dt', '$lib'.split('/')[-1], 'ms %.4f'%d['ms_per_step'], 'GB/s %.0f'%d['value'], 'frac %.3f'%d['roofline']['frac'], [round(r['ms'],4) for r in d['per_round']])"
  done
done
done
timeout 900 python -m pytest tests/test_gpu_fast.py -q -p no:cacheprovider -x 2>&1 | tail -2

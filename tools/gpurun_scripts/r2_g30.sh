# round 2: A/B (1) L2 prefetch of the pass kernel's factor pages (BF_PASS_PF 0 / 2 / 4),
# (2) the tile kernel's compile-time n-tile count (default) vs the branchy k-loop; parity subset
for rep in 1 2; do
for lib in varlibs/libbfapply_pf0.so paper_2007_00202_b200/libbfapply.so varlibs/libbfapply_pf4.so; do
  for dt in c128 c64; do
    BF_LIB=$PWD/$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --dtype $dt > gpurun_out/r2_g30.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/r2_g30.json').read().strip().splitlines()[-1])
print('$dt', '$lib'.split('/')[-1], 'ms %.4f'%d['ms_per_step'], 'GB/s %.0f'%d['value'], 'frac %.3f'%d['roofline']['frac'], [round(r['ms'],4) for r in d['per_round']])"
  done
done
done
for lib in varlibs/libbfapply_branchy.so paper_2007_00202_b200/libbfapply.so; do
  for c in cfg2 cfg3 cfg4; do
    BF_LIB=$PWD/$lib timeout 600 python tools/time_configs.py $c 2>&1 | python -c "
import sys,json
for line in sys.stdin:
    if line.startswith('cfg'):
        k,v=line.split(' ',1); d=json.loads(v); print(k, '$lib'.split('/')[-1], 'N %.4f C %.4f'%(d['N']['ms'], d['C']['ms']), [x['ms'] for x in d['N']['detail']])"
  done
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fast.py -q -p no:cacheprovider -x 2>&1 | tail -2

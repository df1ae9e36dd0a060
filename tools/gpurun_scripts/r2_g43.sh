# round 2: does a deeper page ring pay?  complex128 passes of <= 2 levels with tight windows and a
# 5-page ring (varlibs/libbfapply_tight.so), default plans vs 2-level windows everywhere (BF_C128_DMAX=2)
for rep in 1 2; do
for lib in paper_2007_00202_b200/libbfapply.so varlibs/libbfapply_tight.so; do
  for dm in 3 2; do
    BF_C128_DMAX=$dm BF_LIB=$PWD/$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_g43.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/r2_g43.json').read().strip().splitlines()[-1])
print('$lib'.split('/')[-1], 'dmax=$dm', 'ms %.4f'%d['ms_per_step'], [round(r['ms'],4) for r in d['per_round']])"
  done
done
done
BF_C128_DMAX=2 BF_LIB=$PWD/varlibs/libbfapply_tight.so timeout 900 python -m pytest tests/test_gpu_fast.py -q -p no:cacheprovider -x -k "c128 or complex128" 2>&1 | tail -2

# round 2: A/B the pair-op k-loop order (MMAs before the next page's wait, mid-op releases one k-step
# late; default) vs the previous order (varlibs/libbfapply_order0.so)
timeout 1500 python -m pytest tests/test_gpu_fast.py tests/test_gpu_dist.py tests/test_gpu_fuzz.py -q -p no:cacheprovider -x 2>&1 | tail -2
for rep in 1 2; do
for lib in varlibs/libbfapply_order0.so paper_2007_00202_b200/libbfapply.so; do
  for dt in c128 c64; do
    for nr in 32 8; do
    BF_LIB=$PWD/$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --dtype $dt --nrhs $nr > gpurun_out/r2_g44.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/r2_g44.json').read().strip().splitlines()[-1])
print('$lib'.split('/')[-1], '$dt nrhs=$nr', 'ms %.4f'%d['ms_per_step'], [round(r['ms'],4) for r in d['per_round']])"
    done
  done
done
done

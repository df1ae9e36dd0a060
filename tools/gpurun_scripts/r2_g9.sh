# round 2: deeper ring for nrhs <= 16 (one window half): A/B against the 3/4-page build
for nr in 1 8 16; do
  for dt in c128 c64; do
    for lib in varlibs/libbfapply_np3.so paper_2007_00202_b200/libbfapply.so; do
      BF_LIB=$PWD/$lib python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --dtype $dt --nrhs $nr > gpurun_out/r2_g9.json 2>/dev/null
      python -c "
import json; d=json.loads(open('gpurun_out/r2_g9.json').read().strip().splitlines()[-1])
print('$dt nrhs=$nr', '$lib'.split('/')[-1], 'ms %.4f'%d['ms_per_step'], 'GB/s %.0f'%d['value'], 'frac %.3f'%d['roofline']['frac'], d['roofline']['bound'])"
    done
  done
done
python -m pytest tests/test_gpu_fast.py -x -q -p no:cacheprovider -k "half_tile or large_leaves or layouts" 2>&1 | tail -2

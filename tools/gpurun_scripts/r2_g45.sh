# round 2: generic tile kernels skipping the zero-filled k-steps past a term's K (default) vs running
# every k-step of the chunk (varlibs/libbfapply_nokskip.so); parity of the generic paths
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_extract.py tests/test_gpu_rmatvec.py tests/test_gpu_hinv.py tests/test_gpu_mf.py -q -p no:cacheprovider -x 2>&1 | tail -2
for rep in 1 2; do
for lib in varlibs/libbfapply_nokskip.so paper_2007_00202_b200/libbfapply.so; do
  for c in cfg2 cfg3 cfg4; do
    BF_LIB=$PWD/$lib timeout 600 python tools/time_configs.py $c 2>&1 | python -c "
import sys,json
for line in sys.stdin:
    if line.startswith('cfg'):
        k,v=line.split(' ',1); d=json.loads(v); print(k, '$lib'.split('/')[-1], 'N %.4f C %.4f'%(d['N']['ms'], d['C']['ms']))"
  done
done
done

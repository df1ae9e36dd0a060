# round 2: tile kernels at 3 CTAs / SM (both dtypes, both orientations) vs 2
for mb in 2 3; do
  BF_TILE_MINB=$mb python tools/time_configs.py cfg1 cfg2 cfg3 > gpurun_out/r2_g12_mb$mb.txt 2>&1
  echo "MINB=$mb"; python - <<PY
import json
for line in open("gpurun_out/r2_g12_mb$mb.txt"):
    if line[:3] == "cfg":
        k, j = line.split(" ", 1); d = json.loads(j)
        print(" ", k, "N %.4f C %.4f" % (d["N"]["ms"], d["C"]["ms"]))
PY
  BF_TILE_MINB=$mb python tools/time_configs.py cfg4 2>&1 | python -c "
import sys,json
for line in sys.stdin:
    if line[:3]=='cfg':
        k,j=line.split(' ',1); d=json.loads(j); print(' ', k, 'N %.3f C %.3f'%(d['N']['ms'],d['C']['ms']))"
  BF_TILE_MINB=$mb python tools/time_next.py next4 2>&1 | tail -1 | cut -c1-200
done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_mf.py tests/test_gpu_hinv.py -x -q -p no:cacheprovider -k "not cfg5 and not cfg4" 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3

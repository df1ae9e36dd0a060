# round 2: transposed tile kernel at 3 CTAs / SM (78 registers) vs 2
for mb in 2 3; do
  BF_TILE_MINB=$mb python tools/time_configs.py cfg2 cfg3 > gpurun_out/r2_g11_mb$mb.txt 2>&1
  echo "MINB=$mb"; python - <<PY
import json
for line in open("gpurun_out/r2_g11_mb$mb.txt"):
    if line[:3] == "cfg":
        k, j = line.split(" ", 1); d = json.loads(j)
        print(" ", k, "N %.4f C %.4f" % (d["N"]["ms"], d["C"]["ms"]))
PY
  BF_TILE_MINB=$mb python tools/time_configs.py cfg4 2>&1 | python -c "
import sys,json
for line in sys.stdin:
    if line[:3]=='cfg':
        k,j=line.split(' ',1); d=json.loads(j); print(' ', k, 'N %.3f C %.3f'%(d['N']['ms'],d['C']['ms']))"
done
BF_TILE_MINB=3 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ragged or cfg2 or hodbf or cfg3" 2>&1 | tail -2

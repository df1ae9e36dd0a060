# round 2: transposed tile kernel grid modes (0: item per CTA, 1: unit per CTA, all column tiles)
for g in 0 1; do
  BF_TILE_GRID=$g python tools/time_configs.py cfg2 cfg3 > gpurun_out/r2_g10_grid$g.txt 2>&1
  echo "BF_TILE_GRID=$g"; python - <<PY
import json
for line in open("gpurun_out/r2_g10_grid$g.txt"):
    if line[:3] == "cfg":
        k, j = line.split(" ", 1); d = json.loads(j)
        print(" ", k, "N %.4f C %.4f" % (d["N"]["ms"], d["C"]["ms"]), [x["ms"] for x in d["N"]["detail"]])
PY
  BF_TILE_GRID=$g python tools/time_configs.py cfg4 2>&1 | python -c "
import sys,json
for line in sys.stdin:
    if line[:3]=='cfg':
        k,j=line.split(' ',1); d=json.loads(j); print(' ', k, 'N %.3f C %.3f'%(d['N']['ms'],d['C']['ms']))"
done
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ragged or cfg2 or hodbf or cfg3 or identity or nrhs" 2>&1 | tail -2

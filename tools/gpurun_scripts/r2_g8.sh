for m in 0 1; do
  BF_TILE=$m python tools/time_configs.py cfg2 cfg3 > gpurun_out/r2_g8_tile$m.txt 2>&1
  echo "BF_TILE=$m"; python - <<PY
import json
for line in open("gpurun_out/r2_g8_tile$m.txt"):
    if line[:3] == "cfg":
        k, j = line.split(" ", 1); d = json.loads(j)
        print(" ", k, "N %.4f C %.4f" % (d["N"]["ms"], d["C"]["ms"]), [x["ms"] for x in d["N"]["detail"]])
PY
done
BF_TILE=1 python tools/time_configs.py cfg4 2>&1 | python -c "
import sys,json
for line in sys.stdin:
    if line[:3]=='cfg':
        k,j=line.split(' ',1); d=json.loads(j); print(k, 'N %.3f C %.3f'%(d['N']['ms'],d['C']['ms']))"
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ragged or cfg2 or hodbf or cfg3 or identity" 2>&1 | tail -2

# round 2: generic kernel experiments (transposed orientation, stages)
BF_TILE_T=1 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "ragged or cfg2 or hodbf_small or cfg1 or identity or nrhs_edges or cfg3" > gpurun_out/r2_g6_pytest.log 2>&1
echo "pytest T rc=$?"; tail -3 gpurun_out/r2_g6_pytest.log
for cfg in "0 2" "0 3" "0 4" "1 2" "1 3" "1 4"; do
  set -- $cfg
  BF_TILE_T=$1 BF_TILE_NST=$2 python tools/time_configs.py cfg2 cfg3 > gpurun_out/r2_g6_T$1_N$2.txt 2>&1
  echo "T=$1 NST=$2"; python - <<PY
import json
for line in open("gpurun_out/r2_g6_T$1_N$2.txt"):
    if line[:3] in ("cfg",):
        k, j = line.split(" ", 1); d = json.loads(j)
        print(" ", k, "N %.4f C %.4f" % (d["N"]["ms"], d["C"]["ms"]))
PY
done

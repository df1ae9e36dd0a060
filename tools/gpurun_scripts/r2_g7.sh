# round 2: persistent transposed tile kernel + gemv kernel: parity and timings
python -m pytest tests/test_gpu_parity.py tests/test_gpu_extract.py tests/test_gpu_mf.py tests/test_gpu_hinv.py tests/test_gpu_rmatvec.py -x -q -p no:cacheprovider -k "not cfg5 and not cfg4" > gpurun_out/r2_g7_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r2_g7_pytest.log
for m in 0 1; do
  BF_TILE=$m python tools/time_configs.py cfg1 cfg2 cfg3 > gpurun_out/r2_g7_tile$m.txt 2>&1
  echo "BF_TILE=$m"; python - <<PY
import json
for line in open("gpurun_out/r2_g7_tile$m.txt"):
    if line[:3] == "cfg":
        k, j = line.split(" ", 1); d = json.loads(j)
        print(" ", k, "N %.4f C %.4f" % (d["N"]["ms"], d["C"]["ms"]), [x["ms"] for x in d["N"]["detail"]])
PY
  BF_TILE=$m python tools/time_next.py next4 2>&1 | tail -1
done

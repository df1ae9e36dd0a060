# round 2, re-entry: smoke under an ncu launch list (the driver's round-end check: limit 900 s, 1000 launches) and the widened test_cfg3
mkdir -p gpurun_out/h2
S=$SECONDS
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/h2/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h2/smoke_ncu.log 2>&1; echo "ncu smoke rc $? in $((SECONDS-S)) s"; grep -E "smoke" gpurun_out/h2/smoke_ncu.log | tail -6; wc -l gpurun_out/h2/smoke_launches.csv
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "cfg3" 2>&1 | tail -3

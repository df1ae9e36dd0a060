# round 2: host-apply pipeline on a third stream (apply overlaps the previous D2H), PCIe context,
# default bench line, source-level ncu of the complex64 4-level pass
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "host or graph or streams" 2>&1 | tail -2
timeout 300 python tools/pcie_bw.py
timeout 900 python bench.py > gpurun_out/r2_g29_bench.json 2> gpurun_out/r2_g29_bench.err; echo bench rc $?
python -c "
import json; d=json.loads(open('gpurun_out/r2_g29_bench.json').read().strip().splitlines()[-1])
print('ms %.4f GB/s %.0f e2e %.1f GB/s (%.2f ms)'%(d['ms_per_step'], d['value'], d['e2e']['value'], d['e2e']['ms_per_step']))"
mkdir -p gpurun_out/ev
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bf_pass -s 0 -c 1 -o gpurun_out/ev/src_pass4_c64 python bench.py --dtype c64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu rc $?

# round 2: full GPU suite + smoke + default bench line on the final code (HostPipe, clock ramp)
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_g33_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2_g33_pytest.log; tail -3 gpurun_out/r2_g33_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_g33_smoke.log 2>&1; tail -1 gpurun_out/r2_g33_smoke.log
timeout 900 python bench.py > gpurun_out/r2_g33_bench.json 2> gpurun_out/r2_g33_bench.err; echo bench rc $?
python -c "
import json; d=json.loads(open('gpurun_out/r2_g33_bench.json').read().strip().splitlines()[-1])
print('ms %.4f GB/s %.0f frac %.3f e2e %.1f GB/s (%.2f ms) clocks %s'%(d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['ms_per_step'], d['clocks']))"
timeout 600 python bench.py --nrhs 1 --dtype c64 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_g33_c64n1.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r2_g33_c64n1.json').read().strip().splitlines()[-1])
print('c64 nrhs1 ms %.4f GB/s %.0f e2e %.0f'%(d['ms_per_step'], d['value'], d['e2e']['value']))"

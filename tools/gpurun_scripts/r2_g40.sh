# round 2, final: full GPU suite, smoke, default bench line and the c64 / op C / nrhs lines on the final code
O=gpurun_out/ev5; mkdir -p $O
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_c128.json 2> $O/bench_c128.err
timeout 900 python bench.py --dtype c64 > $O/bench_c64.json 2> $O/bench_c64.err
timeout 600 python bench.py --op C --no-cpu-baseline > $O/bench_c128_C.json 2> /dev/null
for nr in 1 8; do
  timeout 600 python bench.py --nrhs $nr --no-cpu-baseline > $O/bench_c128_nrhs$nr.json 2>/dev/null
  timeout 600 python bench.py --nrhs $nr --dtype c64 --no-cpu-baseline > $O/bench_c64_nrhs$nr.json 2>/dev/null
done
for f in $O/bench_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], 'ms %.4f'%d['ms_per_step'], 'GB/s %.0f'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'e2e %.0f'%d['e2e']['value'], d['clocks']['sm_mhz'])"; done

# round 2, final code: full GPU suite, smoke, default bench line
O=gpurun_out/ev6; mkdir -p $O
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_c128.json 2> $O/bench_c128.err
python -c "
import json; d=json.loads(open('$O/bench_c128.json').read().strip().splitlines()[-1]); print('ms %.4f GB/s %.0f frac %.3f e2e %.0f'%(d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value']), d['clocks'])"

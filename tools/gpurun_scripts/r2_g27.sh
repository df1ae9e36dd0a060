# round 2: P = 8 per-rank compute of the split: complex64 with 3-level vs 4-level windows
for v in 4 3; do
BF_C64_DMAX=$v timeout 300 python tools/time_split.py c64 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('dmax $v single %.4f'%d['single_gpu_ms'], {k:(round(d[k]['max_ms'],4), round(d[k]['eff_vs_single'],3)) for k in ('P1','P2','P4','P8')})"
done

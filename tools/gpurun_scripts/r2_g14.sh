# round 2: fused split exchanging at the pass-minimising level: parity (emulated) + per-rank timing
python -m pytest tests/test_gpu_dist.py -x -q -p no:cacheprovider 2>&1 | tail -2
python tools/time_split.py c128 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('c128', {k:(round(v['max_ms'],4), round(v['eff_vs_single'],3)) for k,v in d.items() if k.startswith('P')})"
BF_DIST_LX=7 python tools/time_split.py c128 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('c128 lx=7', {k:(round(v['max_ms'],4), round(v['eff_vs_single'],3)) for k,v in d.items() if k.startswith('P')})"
python tools/time_split.py c64 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('c64', {k:(round(v['max_ms'],4), round(v['eff_vs_single'],3)) for k,v in d.items() if k.startswith('P')})"

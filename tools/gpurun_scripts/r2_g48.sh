# round 2: transposed tile kernel at 4 CTAs / SM (BF_TILE_MINB=4, 64 registers) vs 3
for rep in 1 2; do
for v in 3 4; do
  for c in cfg2 cfg3 cfg4; do
    BF_TILE_MINB=$v timeout 600 python tools/time_configs.py $c 2>&1 | python -c "
import sys,json
for line in sys.stdin:
    if line.startswith('cfg'):
        k,v=line.split(' ',1); d=json.loads(v); print(k, 'minb=$v', 'N %.4f C %.4f'%(d['N']['ms'], d['C']['ms']))"
  done
done
done

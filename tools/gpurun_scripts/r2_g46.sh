# round 2: configs 1-4 on the final generic kernels (profiles/r02f_configs.txt)
timeout 1500 python tools/time_configs.py cfg1 cfg2 cfg3 cfg4 > gpurun_out/r2_g46_configs.txt 2> gpurun_out/r2_g46_configs.err
python -c "
import json
for line in open('gpurun_out/r2_g46_configs.txt'):
    if line.startswith('cfg'):
        k,v=line.split(' ',1); d=json.loads(v); print(k, 'N %.4f C %.4f graph %.4f'%(d['N']['ms'], d['C']['ms'], d['N']['ms_graph']))"

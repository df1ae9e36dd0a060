# round 2, re-entry: leaf kernels with 12 / 16 item-owning warps per CTA (BF_LEAF_NW_IN / _OUT) against 8,
# with the chunk sizes (BF_LEAF_KC / BF_LEAF_MC) that keep the per-warp stage depth
run() {  # label, dtype
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --dtype $2 > gpurun_out/r2_h4.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2_h4.json').read().strip().splitlines()[-1])
pr=d['per_round']; print('$2 $1', 'ms %.4f'%d['ms_per_step'], 'leaf-in %.4f'%pr[0]['ms'], 'last %s %.4f'%(pr[-1]['kernel'], pr[-1]['ms']))"
}
for rep in 1 2; do
  unset BF_LEAF_NW_IN BF_LEAF_NW_OUT BF_LEAF_KC BF_LEAF_MC
  run "nw 8/8 default" c64
  BF_LEAF_NW_IN=12 BF_LEAF_NW_OUT=12 run "nw 12/12 kc32 mc64" c64
  BF_LEAF_NW_IN=12 BF_LEAF_NW_OUT=12 BF_LEAF_KC=16 BF_LEAF_MC=32 run "nw 12/12 kc16 mc32" c64
  BF_LEAF_NW_IN=16 BF_LEAF_NW_OUT=16 BF_LEAF_KC=16 BF_LEAF_MC=32 run "nw 16/16 kc16 mc32" c64
  BF_LEAF_NW_IN=16 BF_LEAF_NW_OUT=16 run "nw 16/16 kc32 mc64" c64
  BF_LEAF_NW_IN=16 BF_LEAF_NW_OUT=16 BF_LEAF_KC=16 BF_LEAF_MC=16 run "nw 16/16 kc16 mc16" c64
  run "nw 8 default" c128
  BF_LEAF_NW_IN=12 run "nw 12 kc16" c128
  BF_LEAF_NW_IN=12 BF_LEAF_KC=8 run "nw 12 kc8" c128
  BF_LEAF_NW_IN=16 run "nw 16 kc16" c128
done
for nw in 12 16; do
  BF_LEAF_NW_IN=$nw BF_LEAF_NW_OUT=$nw BF_LEAF_KC=16 BF_LEAF_MC=32 timeout 900 python -m pytest tests/test_gpu_fast.py -q -p no:cacheprovider -x -k "layouts or large_leaves" 2>&1 | tail -1
done

#!/bin/bash
# complex64 pass: window buffers x ring pages A/B on one box (variant libraries in varlibs/)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/r3k.txt; : > $out
LIB=paper_2007_00202_b200/libbfapply.so
cp $LIB /tmp/lib_orig.so
for rep in 1 2; do
for v in w2_p4 w3_p4 w2_p5 w3_p3; do
  cp varlibs/lib_$v.so $LIB
  r=$(timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --dtype c64 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);r=d['per_round'];print(round(d['ms_per_step'],4),[round(x['ms'],4) for x in r])")
  echo "$v: $r" >> $out
done; done
cp /tmp/lib_orig.so $LIB
echo done

# round 2: level-wise extraction in one cooperative launch (vs per-stage launches, vs the compact plan)
python -m pytest tests/test_gpu_extract.py tests/test_gpu_hinv.py -x -q -p no:cacheprovider 2>&1 | tail -3
BF_EXTRACT_TIMING=1 python tools/time_extract.py c128 > gpurun_out/r2_extract6.txt 2> gpurun_out/r2_extract6_timing.txt
tail -1 gpurun_out/r2_extract6.txt | cut -c1-900
sed -n '2p;14p;20p;26p;32p;38p;44p' gpurun_out/r2_extract6_timing.txt
BF_XLEVEL_STAGES=1 python tools/time_extract.py c128 2>/dev/null | tail -1 | cut -c1-900
BF_EXTRACT_COMPACT=1 python tools/time_extract.py c128 2>/dev/null | tail -1 | cut -c1-900

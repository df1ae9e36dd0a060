# round 2: level-wise extraction, 8-row chunks per thread
python -m pytest tests/test_gpu_extract.py tests/test_gpu_hinv.py tests/test_gpu_rmatvec.py tests/test_gpu_mf.py -x -q -p no:cacheprovider 2>&1 | tail -3
BF_EXTRACT_TIMING=1 python tools/time_extract.py c128 > gpurun_out/r2_extract5.txt 2> gpurun_out/r2_extract5_timing.txt
tail -1 gpurun_out/r2_extract5.txt | cut -c1-900
grep 8097792 gpurun_out/r2_extract5_timing.txt | tail -2; grep "327 parts" gpurun_out/r2_extract5_timing.txt | tail -2
BF_EXTRACT_COMPACT=1 python tools/time_extract.py c128 2>/dev/null | tail -1 | cut -c1-900

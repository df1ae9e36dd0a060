# round 2: compact extraction planner in parallel (host thread pool) + pinned table upload
python -m pytest tests/test_gpu_extract.py -x -q -p no:cacheprovider 2>&1 | tail -2
BF_EXTRACT_TIMING=1 python tools/time_extract.py c128 > gpurun_out/r2_extract2.txt 2> gpurun_out/r2_extract2_timing.txt
tail -3 gpurun_out/r2_extract2.txt | cut -c1-600
grep -c . gpurun_out/r2_extract2_timing.txt; sed -n '13,18p' gpurun_out/r2_extract2_timing.txt
nproc

# round 2: level-wise extraction (products enumerated on the device)
python -m pytest tests/test_gpu_extract.py -x -q -p no:cacheprovider 2>&1 | tail -5
BF_EXTRACT_TIMING=1 python tools/time_extract.py c128 > gpurun_out/r2_extract4.txt 2> gpurun_out/r2_extract4_timing.txt
tail -1 gpurun_out/r2_extract4.txt | cut -c1-900
sort gpurun_out/r2_extract4_timing.txt | uniq -c | sort -rn | head -12

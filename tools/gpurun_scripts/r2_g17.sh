# round 2: extraction timing breakdown (host threads 16 vs 1)
BF_EXTRACT_TIMING=1 python tools/time_extract.py c128 > gpurun_out/r2_extract3.txt 2> gpurun_out/r2_extract3_timing.txt
BF_HOST_THREADS=1 BF_EXTRACT_TIMING=1 python tools/time_extract.py c128 > gpurun_out/r2_extract3_t1.txt 2> gpurun_out/r2_extract3_t1_timing.txt
sed -n '13,18p' gpurun_out/r2_extract3_timing.txt; sed -n '13,18p' gpurun_out/r2_extract3_t1_timing.txt
tail -1 gpurun_out/r2_extract3.txt | cut -c1-500; tail -1 gpurun_out/r2_extract3_t1.txt | cut -c1-500

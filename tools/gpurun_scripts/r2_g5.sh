# round 2: timings of NEXT-2/3/4
python tools/time_next.py > gpurun_out/r2_time_next.jsonl 2> gpurun_out/r2_time_next.err
echo "rc=$?"
cat gpurun_out/r2_time_next.jsonl; tail -5 gpurun_out/r2_time_next.err

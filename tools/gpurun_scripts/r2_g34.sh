# round 2: the solve sweep (NEXT-4) with concurrent fronts per height / depth vs the serial sweep
timeout 900 python -m pytest tests/test_gpu_mf.py tests/test_gpu_hinv.py -q -p no:cacheprovider 2>&1 | tail -2
for lib in varlibs/libbfapply_mfserial.so paper_2007_00202_b200/libbfapply.so; do
  echo $lib; BF_LIB=$PWD/$lib timeout 900 python tools/time_next.py next4 2>/dev/null | cut -c1-600
done

mkdir -p gpurun_out
for lib in libsdme_pref00.so libsdme.so libsdme_pref21.so; do
 for var in 0 14; do
  echo "== $lib variant $var"
  SDME_LIB=paper_2104_13466_b200/$lib SDME_VARIANT=$var timeout 300 python tools/op_times.py 2>&1 | tail -1
 done
done
SDME_LIB=paper_2104_13466_b200/libsdme.so timeout 600 python tools/q5_check.py 14 12 2>&1 | grep -v "bit-identical" | tail -20
SDME_LIB=paper_2104_13466_b200/libsdme_pref21.so timeout 600 python tools/q5_check.py 14 12 2>&1 | grep -v "bit-identical" | tail -20
SDME_LIB=paper_2104_13466_b200/libsdme.so timeout 300 python tools/pcg_iter_time.py 64 4 5 2>&1 | head -1
SDME_LIB=paper_2104_13466_b200/libsdme.so SDME_VARIANT=14 timeout 300 python tools/pcg_iter_time.py 64 4 5 2>&1 | head -1

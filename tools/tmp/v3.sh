for lib in libsdme_pref31.so libsdme_pref42.so; do
 for var in 0 14; do
  echo "== $lib variant $var"
  SDME_LIB=paper_2104_13466_b200/$lib SDME_VARIANT=$var timeout 300 python tools/op_times.py 2>&1 | tail -1
 done
 SDME_LIB=paper_2104_13466_b200/$lib timeout 600 python tools/q5_check.py 14 12 2>&1 | grep -v "bit-identical" | tail -20
done

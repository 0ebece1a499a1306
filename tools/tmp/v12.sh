for lib in libsdme_nobox.so libsdme.so libsdme_nobox.so libsdme.so; do
  echo "== $lib"
  SDME_LIB=paper_2104_13466_b200/$lib timeout 300 python tools/op_times.py 2>&1 | tail -1
  for P in 3 6; do SDME_LIB=paper_2104_13466_b200/$lib timeout 300 python tools/kp_p.py $P 2>&1 | tail -1; done
done
for lib in libsdme_nogeo.so libsdme.so; do
  echo "== $lib"
  SDME_LIB=paper_2104_13466_b200/$lib timeout 600 python tools/gen_mesh_bench.py 32 48 2>&1 | cut -c1-420
done

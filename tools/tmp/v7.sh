for g in 0 1 3 4 5 7; do echo "PCG_CHAIN $g";
SDME_PCG_CHAIN=$g timeout 300 python tools/pcg_iter_time.py 64 4 5 2>&1 | cut -c1-200
SDME_PCG_CHAIN=$g timeout 600 python tools/run_configs.py c5:-1.3e6:SDME_H 2>&1 | cut -c1-130
done

for g in 0 1; do echo "PCG_CHAIN $g";
SDME_PCG_CHAIN=$g timeout 300 python tools/pcg_iter_time.py 64 4 5 2>&1
SDME_PCG_CHAIN=$g timeout 600 python tools/run_configs.py c5:-1.3e6:SDME_H 2>&1 | cut -c1-300
done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/q5_check.py 2>&1 | grep -v "bit-identical" | tail

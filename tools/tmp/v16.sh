for g in 5 9 5 9; do echo "PCG_CHAIN $g";
SDME_PCG_CHAIN=$g timeout 300 python tools/pcg_iter_time.py 64 4 5 2>&1 | cut -c1-200
SDME_PCG_CHAIN=$g timeout 300 python tools/prof_pcg_c5.py --time 2>&1 | grep "per iteration"
done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3

for g in 0 1; do echo "GRAPH_PDL $g";
SDME_GRAPH_PDL=$g timeout 300 python tools/pcg_iter_time.py 64 4 5 2>&1
SDME_GRAPH_PDL=$g timeout 600 python tools/run_configs.py c5:-1.3e6:SDME_H 2>&1 | cut -c1-300
done
SDME_GRAPH_PDL=1 timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3

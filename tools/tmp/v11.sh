for pdl in 0 1; do echo "SDME_PDL=$pdl"; SDME_PDL=$pdl timeout 600 python tools/run_configs.py c1 2>&1 | cut -c1-120; SDME_PDL=$pdl timeout 300 python tools/pcg_iter_time.py 4 4 6 2>&1 | head -1 | cut -c1-200; done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3

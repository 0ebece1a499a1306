timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/pcg_iter_time.py 64 4 5 2>&1 | cut -c1-200
timeout 300 python tools/prof_pcg_c5.py --time 2>&1 | grep "per iteration"
timeout 900 python tools/run_configs.py c1 c5 2>&1 | cut -c1-140

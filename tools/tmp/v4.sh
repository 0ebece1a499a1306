for sl in 1 2 4 8; do echo "slabs $sl"; SDME_SLABS=$sl timeout 300 python tools/op_times.py 2>&1 | tail -1; done
timeout 300 python tools/pcg_iter_time.py 64 4 5 2>&1
timeout 600 python tools/q5_check.py 2>&1 | grep -v "bit-identical" | tail
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 1200 python tools/run_configs.py c1 c5 2>&1 | cut -c1-400

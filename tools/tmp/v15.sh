for s in 0 1; do echo "SDME_CONTACT_SIDE=$s"; SDME_CONTACT_SIDE=$s timeout 600 python tools/prof_c4.py 2>&1 | grep "per step"; SDME_CONTACT_SIDE=$s timeout 600 python tools/run_configs.py c4 2>&1 | cut -c1-200; done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3

for s in 0 1 0 1; do echo "SDME_CONTACT_SIDE=$s"; SDME_CONTACT_SIDE=$s timeout 600 python tools/prof_c4.py 2>&1 | grep "per step"; done
timeout 900 python -m pytest tests -m gpu -x -q -k "explicit or contact or impact" 2>&1 | tail -3

for ev in 0 1; do echo "SDME_EV=$ev"; SDME_EV=$ev timeout 600 python tools/prof_c4.py 2>&1 | grep "per step"; done

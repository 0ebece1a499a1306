# config-1 launch list with the PCG iterations as plain launches (SDME_PCG_DIRECT)
SDME_PCG_DIRECT=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1_direct.csv python tools/c1_launches.py 1 > /dev/null 2>&1

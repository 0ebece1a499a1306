timeout 300 python tools/prof_pcg_c5.py --time 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python tools/prof_pcg_c5.py > gpurun_out/c5_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/c5_launches.csv 2>&1 | head -24

timeout 600 python tools/prof_c4.py 2>&1 | tail -3
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python tools/prof_c4.py > gpurun_out/c4_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/c4_launches.csv 2>&1 | head -30
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/q5_check.py 2>&1 | grep -v "bit-identical" | tail -3

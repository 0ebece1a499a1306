mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python tools/op_times.py > gpurun_out/op_times.log 2>&1
timeout 300 python tools/pcg_iter_time.py 64 4 5 > gpurun_out/pcg_iter.log 2>&1
timeout 2400 python tools/run_configs.py c1 c4 c5 --cpu > gpurun_out/configs_145.jsonl 2> gpurun_out/configs_145.err
SDME_LIB=paper_2104_13466_b200/libsdme_checked.so timeout 900 python tools/sanitize_cases.py > gpurun_out/checked_cases.log 2>&1; echo "exit $?" >> gpurun_out/checked_cases.log
SDME_LIB=paper_2104_13466_b200/libsdme_checked.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/checked_pytest.log 2>&1; echo "exit $?" >> gpurun_out/checked_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log

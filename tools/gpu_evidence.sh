# Round evidence on one B200: GPU tests, smoke, bench (ours + reference arm),
# the bench's ncu launch list, per-launch DRAM traffic of K.p / mass / f_int,
# and one ncu --set full capture of the K.p kernel.  Outputs in gpurun_out/.
set -x
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -k regex:element_col -c 24 --csv --log-file gpurun_out/traffic.csv python tools/prof_variant.py > gpurun_out/ncu_traffic.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:element_col -c 1 -o gpurun_out/kp -f python tools/prof_apply.py > gpurun_out/ncu_full.log 2>&1
timeout 1500 python tools/run_configs.py c1 c3 c4 c5 --cpu > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
timeout 600 python tools/gen_mesh_bench.py 32 48 > gpurun_out/gen_mesh.jsonl 2> gpurun_out/gen_mesh.err
# checked build (device bounds / alignment asserts; compute-sanitizer is closed on this pool)
SDME_LIB=paper_2104_13466_b200/libsdme_checked.so timeout 900 python tools/sanitize_cases.py > gpurun_out/checked_cases.log 2>&1; echo "exit $?" >> gpurun_out/checked_cases.log
SDME_LIB=paper_2104_13466_b200/libsdme_checked.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/checked_pytest.log 2>&1; echo "exit $?" >> gpurun_out/checked_pytest.log

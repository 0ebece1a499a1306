# Round evidence on one B200: GPU tests, smoke, bench (ours + reference arm),
# the bench's ncu launch list, per-launch DRAM traffic of K.p / mass / f_int,
# ncu --set full captures of the K.p kernel and of the PCG-side operators
# (setup, stored-data K.p, Jacobi diagonal), config sweeps with the reference's
# CPU path beside them, general meshes, and the checked build.
# Outputs in gpurun_out/.  Every ncu pass follows a plain run of the same
# program that exited 0.
set -x
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python tools/op_times.py > gpurun_out/op_times.log 2>&1
timeout 300 python tools/pcg_iter_time.py 64 4 5 > gpurun_out/pcg_iter.log 2>&1
timeout 300 python tools/q5_check.py > gpurun_out/q5_check.log 2>&1
timeout 300 python tools/q5d_check.py > gpurun_out/q5d_check.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -k regex:element_q5 -c 160 --csv --log-file gpurun_out/traffic.csv python tools/prof_variant.py > gpurun_out/ncu_traffic.log 2>&1
# one colour pass of 32,768 elements (SDME_SLABS=1: the default z-slab schedule splits it in 8)
SDME_SLABS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:element_q5 -s 8 -c 1 -o gpurun_out/kp -f python tools/prof_apply.py > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none -k "regex:element_q5|element_col" -c 17 -o gpurun_out/pcg_ops -f python tools/prof_pcg_ops.py > gpurun_out/ncu_pcg_ops.log 2>&1
# summaries on the box; the reports themselves are too large to bring back (64 MiB cap)
python tools/ncu_summary.py gpurun_out/kp.ncu-rep > gpurun_out/ncu_kp_summary.txt 2>&1
python tools/ncu_sass_ops.py gpurun_out/kp.ncu-rep > gpurun_out/ncu_kp_sassops.txt 2>&1
python tools/ncu_summary.py gpurun_out/pcg_ops.ncu-rep > gpurun_out/ncu_pcg_ops_summary.txt 2>&1
rm -f gpurun_out/pcg_ops.ncu-rep gpurun_out/kp.ncu-rep
timeout 2400 python tools/run_configs.py c1 c3 c4 c5 --cpu > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
timeout 600 python tools/gen_mesh_bench.py 32 48 > gpurun_out/gen_mesh.jsonl 2> gpurun_out/gen_mesh.err
# checked build (device bounds / alignment asserts; compute-sanitizer is closed on this pool)
SDME_LIB=paper_2104_13466_b200/libsdme_checked.so timeout 900 python tools/sanitize_cases.py > gpurun_out/checked_cases.log 2>&1; echo "exit $?" >> gpurun_out/checked_cases.log
SDME_LIB=paper_2104_13466_b200/libsdme_checked.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/checked_pytest.log 2>&1; echo "exit $?" >> gpurun_out/checked_pytest.log

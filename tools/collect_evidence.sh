# Copy the outputs of tools/gpu_evidence.sh (gpurun_out/ or the directory given) into
# profiles/ under this round's names.   bash tools/collect_evidence.sh [dir] [round]
set -e
src=${1:-gpurun_out}
r=${2:-r02}
cp $src/bench.json profiles/bench_$r.json
cp $src/bench_ref.json profiles/bench_${r}_reference.json
cp $src/launches.csv profiles/ncu_launches_$r.csv
python tools/launch_summary.py $src/launches.csv > profiles/ncu_launches_${r}_summary.txt
python tools/ncu_traffic.py $src/traffic.csv profiles/ncu_traffic_$r.json
cat $src/ncu_kp_summary.txt $src/ncu_kp_sassops.txt > profiles/ncu_apply_$r.txt
cp $src/ncu_pcg_ops_summary.txt profiles/ncu_pcg_ops_$r.txt
grep '^{' $src/configs.jsonl > profiles/configs_$r.jsonl
grep '^{' $src/gen_mesh.jsonl > profiles/gen_mesh_$r.jsonl
{ echo "tools/op_times.py (ms per call at config 2; '+m': with the mass term c_m = 4e8)"; cat $src/op_times.log; echo;
  echo "tools/pcg_iter_time.py 64 4 5 (Jacobi-PCG, c_m = 4e8)"; cat $src/pcg_iter.log; } > profiles/op_times_$r.txt
cat $src/q5_check.log $src/q5d_check.log > profiles/q5_check_$r.log
cp $src/checked_cases.log profiles/checked_build_cases_$r.log
cp $src/checked_pytest.log profiles/checked_build_pytest_$r.log
tail -3 $src/pytest_gpu.log > profiles/pytest_gpu_$r.log
tail -2 $src/smoke.log >> profiles/pytest_gpu_$r.log

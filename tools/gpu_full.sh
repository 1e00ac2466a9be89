# Full round-end evidence on one B200 (run under gpurun): GPU tests, smoke,
# bench (default + reference arm + other workloads), launch list and
# `ncu --set full` of the two top kernels.  Everything lands in
# gpurun_out/${TAG}_*.
# usage: bash tools/gpu_full.sh TAG
TAG=${1:-full}
O=gpurun_out/${TAG}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > ${O}_gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > ${O}_pytest_gpu.log 2>&1; echo "pytest=$?" >> ${O}_status.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; echo "smoke=$?" >> ${O}_status.txt
timeout 900 python bench.py > ${O}_bench_default.json 2> ${O}_bench_default.err; echo "bench=$?" >> ${O}_status.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > ${O}_bench_reference.json 2> ${O}_bench_reference.err; echo "reference=$?" >> ${O}_status.txt
for w in allegro_cylinder leap_mug leap_hammer leap_drill four_finger_sphere; do
  timeout 600 python bench.py --no-cpu --workload $w --steps 3 --warmup 3 2>/dev/null | tail -1 >> ${O}_bench_other.jsonl
done
timeout 600 python bench.py --no-cpu --workload leap_mug --batch 12500 --steps 3 --warmup 3 2>/dev/null | tail -1 >> ${O}_bench_other.jsonl
timeout 900 python bench.py --no-cpu --workload shadow_icosphere --batch 2000 --steps 3 --warmup 3 2>/dev/null | tail -1 >> ${O}_bench_other.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 150 --csv --log-file ${O}_launches.csv \
  python bench.py --no-cpu --no-clocks --steps 1 --warmup 3 > ${O}_ncu_launches.log 2>&1
python tools/launch_summary.py ${O}_launches.csv > ${O}_launch_summary.txt
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_contact_opt2|k_realize_warp|k_collision3" -c 3 \
  -o ${O}_full -f python bench.py --no-cpu --no-clocks --steps 1 --warmup 1 > ${O}_ncu_full.log 2>&1
echo "ncu_full=$?" >> ${O}_status.txt

# parity + A/B of the realize launch bound + launch list
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for mb in 4 5; do export LG_COPT_MINB=$mb
  python bench.py --no-cpu --steps 5 --warmup 3 > gpurun_out/bench_mb$mb.log 2>&1; echo "mb=$mb rc=$?"
  tail -1 gpurun_out/bench_mb$mb.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["stage_seconds"], d["work"])'
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --no-cpu --no-clocks --steps 1 --warmup 3 > gpurun_out/ncu_l.log 2>&1; python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt; head -6 gpurun_out/launch_summary.txt

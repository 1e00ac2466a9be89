# parity + A/B of a launch-bound env knob ($AB_VAR over $AB_VALS) + launch list
AB_VAR=${AB_VAR:-LG_REALIZE_MINB}; AB_VALS=${AB_VALS:-"5 6"}
timeout 600 python -m pytest tests -m gpu -x -q --timeout=300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for v in $AB_VALS; do export $AB_VAR=$v
  timeout 300 python bench.py --no-cpu --steps 5 --warmup 3 > gpurun_out/bench_ab$v.log 2>&1; echo "$AB_VAR=$v rc=$?"
  tail -1 gpurun_out/bench_ab$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["stage_seconds"])'
done
unset $AB_VAR
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --no-cpu --no-clocks --steps 1 --warmup 3 > gpurun_out/ncu_l.log 2>&1; python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt; head -6 gpurun_out/launch_summary.txt

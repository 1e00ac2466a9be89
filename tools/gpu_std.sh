python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
python bench.py --no-cpu --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench.log | cut -c1-300
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --no-cpu --no-clocks --steps 1 --warmup 3 > gpurun_out/ncu_l.log 2>&1; python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt; head -9 gpurun_out/launch_summary.txt

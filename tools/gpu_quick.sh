# Quick device check: parity vs the compiled reference + launch list of the bench pass.
# usage (on the GPU box): bash tools/gpu_quick.sh TAG [pytest -k expr]
TAG=${1:-q}; K=${2:-}
if [ -n "$K" ]; then timeout 900 python -m pytest tests -m gpu -q -x -k "$K" 2>&1 | tail -3 > gpurun_out/${TAG}_tests.log; fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --no-cpu --no-clocks --steps 1 --warmup 3 > gpurun_out/${TAG}_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launch_summary.txt

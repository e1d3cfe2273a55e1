# Quick GPU iteration: selected tests + C2 bench (no CPU baseline).  Usage: bash tools/gpu_quick.sh "<pytest -k expr>"
set -x
K=${1:-aca}
timeout 900 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/pytest_quick.log 2>&1; tail -15 gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-baseline 0 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; tail -c 1500 gpurun_out/bench_quick.json; tail -5 gpurun_out/bench_quick.err

# Round-2 re-entry baseline: smoke, GPU suite, C2 bench, C3 recompute trace.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | grep "Model name"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2a.log 2>&1; tail -2 gpurun_out/smoke_r2a.log
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu_r2a.log 2>&1; tail -22 gpurun_out/pytest_gpu_r2a.log
timeout 900 python bench.py --steps 20 --warmup 3 --cpu-baseline 0 > gpurun_out/bench_c2_r2a.json 2> gpurun_out/bench_c2_r2a.err; tail -c 1500 gpurun_out/bench_c2_r2a.json
HM_TRACE=1 timeout 1200 python bench.py --n 4194304 --d 3 --kernel matern --mode recompute --steps 1 --warmup 1 --cpu-baseline 0 > gpurun_out/bench_c3_r2a.json 2> gpurun_out/bench_c3_r2a.err; tail -c 800 gpurun_out/bench_c3_r2a.json; grep -E "classes|NW|cluster|big|chunk" gpurun_out/bench_c3_r2a.err | tail -30

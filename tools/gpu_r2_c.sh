set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2c.log 2>&1; tail -2 gpurun_out/smoke_r2c.log
timeout 2400 python -m pytest tests -m gpu -q -x --durations=20 > gpurun_out/pytest_gpu_r2c.log 2>&1; tail -30 gpurun_out/pytest_gpu_r2c.log
timeout 900 python bench.py --steps 20 --warmup 3 --cpu-baseline 0 > gpurun_out/bench_c2_r2c.json 2> gpurun_out/bench_c2_r2c.err; tail -c 1500 gpurun_out/bench_c2_r2c.json; tail -3 gpurun_out/bench_c2_r2c.err
HM_TRACE=1 timeout 1200 python bench.py --n 4194304 --d 3 --kernel matern --mode recompute --steps 1 --warmup 1 --cpu-baseline 0 > gpurun_out/bench_c3_r2c.json 2> gpurun_out/bench_c3_r2c.err; tail -c 1500 gpurun_out/bench_c3_r2c.json; grep -E "classes|NW|cluster|big|chunk" gpurun_out/bench_c3_r2c.err | tail -12

set -x
timeout 600 python -m pytest tests/test_gpu_round2.py -m gpu -q -x -k "graph or caller or invariant" > gpurun_out/pytest_r2o.log 2>&1; tail -2 gpurun_out/pytest_r2o.log
timeout 1200 python bench.py --n 4194304 --d 3 --kernel matern --mode recompute --steps 2 --warmup 1 --cpu-baseline 0 > gpurun_out/bench_c3_r2o.json 2> gpurun_out/bench_c3_r2o.err; tail -c 250 gpurun_out/bench_c3_r2o.json
HM_ACA_1STREAM=1 timeout 1200 python bench.py --n 4194304 --d 3 --kernel matern --mode recompute --steps 2 --warmup 1 --cpu-baseline 0 > gpurun_out/bench_c3_r2o1.json 2> gpurun_out/bench_c3_r2o1.err; tail -c 250 gpurun_out/bench_c3_r2o1.json
timeout 1500 python bench.py --n 4194304 --d 4 --kernel gaussian --mode recompute --steps 1 --warmup 1 > gpurun_out/bench_c5g_r2o.json 2> gpurun_out/bench_c5g_r2o.err; tail -c 250 gpurun_out/bench_c5g_r2o.json

# bench lines for the recompute-mode BASELINE configs (parity configs; not the headline)
set -x
timeout 1200 python bench.py --n 4194304 --d 3 --kernel matern --mode recompute --steps 2 --warmup 1 --cpu-baseline 0 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 1200 gpurun_out/bench_c3.json; tail -3 gpurun_out/bench_c3.err
timeout 1200 python bench.py --n 4194304 --d 4 --kernel gaussian --mode recompute --steps 2 --warmup 1 --cpu-baseline 0 > gpurun_out/bench_c5g.json 2> gpurun_out/bench_c5g.err; tail -c 1200 gpurun_out/bench_c5g.json; tail -3 gpurun_out/bench_c5g.err

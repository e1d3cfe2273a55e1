# Final round-1 evidence: full GPU suite, C2 bench (+CPU baseline), reference arm, launch list,
# ncu captures of the product kernels, recompute-config bench lines.
set -x
bash tools/gpu_round.sh r1d
timeout 1500 python bench.py --n 4194304 --d 3 --kernel matern --mode recompute --steps 2 --warmup 1 --cpu-baseline 0 > gpurun_out/bench_c3_r1d.json 2> gpurun_out/bench_c3_r1d.err; tail -c 300 gpurun_out/bench_c3_r1d.json
timeout 1500 python bench.py --n 4194304 --d 4 --kernel gaussian --mode recompute --steps 2 --warmup 1 --cpu-baseline 0 > gpurun_out/bench_c5g_r1d.json 2> gpurun_out/bench_c5g_r1d.err; tail -c 300 gpurun_out/bench_c5g_r1d.json
timeout 600 python tools/bench_multi.py --n 262144 --d 4 --mode recompute --nrhs 16 --steps 2 > gpurun_out/multi_c5s_r1d.jsonl 2>&1; tail -2 gpurun_out/multi_c5s_r1d.jsonl

set -x
timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/bench_c2_r2s.json 2> gpurun_out/bench_c2_r2s.err; tail -c 700 gpurun_out/bench_c2_r2s.json
bash tools/gpu_r2_ncu.sh r2s
timeout 1500 python tools/c5_cg.py 4194304 4 10 exact > gpurun_out/c5cg_r2s.log 2>&1; tail -1 gpurun_out/c5cg_r2s.log | cut -c 1-1500

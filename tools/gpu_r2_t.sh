set -x
timeout 900 python bench.py --steps 30 --warmup 3 --cpu-baseline 0 > gpurun_out/bench_c2_r2t.json 2> gpurun_out/bench_c2_r2t.err; tail -c 400 gpurun_out/bench_c2_r2t.json
timeout 900 ncu -f --metrics gpu__time_duration.sum --clock-control none --csv python tools/multi_once.py 1048576 4 > gpurun_out/multi_launch_exact_r2t.csv 2>/dev/null; tail -2 gpurun_out/multi_launch_exact_r2t.csv | cut -c 1-200
timeout 900 ncu -f --metrics gpu__time_duration.sum --clock-control none --csv python tools/multi_once.py 1048576 4 dmma > gpurun_out/multi_launch_dmma_r2t.csv 2>/dev/null
timeout 600 python tools/bench_multi.py --n 1048576 --d 4 --mode recompute --nrhs 16 --steps 2 > gpurun_out/multi_2e20_r2t.jsonl 2>&1; tail -3 gpurun_out/multi_2e20_r2t.jsonl

set -x
HM_TRACE=1 timeout 600 python tools/setup_time.py 1048576 2 gaussian stored 3 > gpurun_out/setup_c2_r2dd.log 2>&1; grep -v "class [0-9]" gpurun_out/setup_c2_r2dd.log | tail -40
timeout 900 python bench.py --steps 10 --warmup 3 --cpu-baseline 0 > gpurun_out/bench_c2_r2dd.json 2> gpurun_out/bench_c2_r2dd.err; tail -c 600 gpurun_out/bench_c2_r2dd.json

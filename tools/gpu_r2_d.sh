# compaction + stream fix check, C2 bench, ncu full of the ACA kernels (C3-like and C5-like)
set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "stored or aca or graph or c1 or factors or bench_config or caller or timings" > gpurun_out/pytest_r2d.log 2>&1; tail -5 gpurun_out/pytest_r2d.log
timeout 900 python bench.py --steps 30 --warmup 3 --cpu-baseline 0 > gpurun_out/bench_c2_r2d.json 2> gpurun_out/bench_c2_r2d.err; tail -c 1800 gpurun_out/bench_c2_r2d.json; tail -3 gpurun_out/bench_c2_r2d.err
bash tools/ncu_aca_r2.sh aca_m3 1048576 3 matern 'aca_' 0 8
bash tools/ncu_aca_r2.sh aca_g4 262144 4 gaussian 'aca_' 0 8

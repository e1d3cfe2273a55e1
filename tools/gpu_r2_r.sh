set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=12 > gpurun_out/pytest_gpu_r2r.log 2>&1; tail -16 gpurun_out/pytest_gpu_r2r.log
timeout 900 python tools/setup_time.py 16777216 3 gaussian recompute 2 > gpurun_out/setup_c4_r2r.log 2>&1; tail -1 gpurun_out/setup_c4_r2r.log
timeout 600 python tools/setup_time.py 4194304 4 gaussian recompute 2 > gpurun_out/setup_c5_r2r.log 2>&1; tail -1 gpurun_out/setup_c5_r2r.log
timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/bench_c2_r2r.json 2> gpurun_out/bench_c2_r2r.err; tail -c 600 gpurun_out/bench_c2_r2r.json

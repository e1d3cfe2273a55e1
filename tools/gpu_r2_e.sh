# ACA paired-evaluation check: parity subset, C3 recompute bench + trace, d=4 Gaussian trace, C2 build
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_round2.py -m gpu -q -x -k "not config5 and not engine" > gpurun_out/pytest_r2e.log 2>&1; tail -4 gpurun_out/pytest_r2e.log
HM_TRACE=1 timeout 1200 python bench.py --n 4194304 --d 3 --kernel matern --mode recompute --steps 1 --warmup 1 --cpu-baseline 0 > gpurun_out/bench_c3_r2e.json 2> gpurun_out/bench_c3_r2e.err; tail -c 1200 gpurun_out/bench_c3_r2e.json; grep -E "classes|NW|cluster|big|chunk" gpurun_out/bench_c3_r2e.err | tail -10
HM_TRACE=1 timeout 900 python tools/trace_recompute.py 1048576 4 gaussian > gpurun_out/trace_g4_r2e.log 2>&1; grep -E "classes|NW|cluster|big|chunk|mvp|\{" gpurun_out/trace_g4_r2e.log | tail -14
HM_TRACE=1 timeout 600 python tools/trace_build.py > gpurun_out/trace_c2_r2e.log 2>&1; tail -14 gpurun_out/trace_c2_r2e.log

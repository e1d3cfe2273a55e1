set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "aca or mvp_matches" > gpurun_out/pytest_r2l.log 2>&1; tail -3 gpurun_out/pytest_r2l.log
HM_SMOOTH=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_round2.py -m gpu -q -x -k "aca or mvp_matches or c1 or graph or invariant" > gpurun_out/pytest_r2l1.log 2>&1; tail -3 gpurun_out/pytest_r2l1.log
HM_TRACE=1 timeout 900 python tools/trace_recompute.py 1048576 4 gaussian > gpurun_out/trace_g4_r2l.log 2>&1; grep -E "smooth|cluster|big \(|'aca'" gpurun_out/trace_g4_r2l.log | tail -8
HM_TRACE=1 timeout 900 python tools/trace_recompute.py 1048576 3 matern > gpurun_out/trace_m3_r2l.log 2>&1; grep -E "smooth|cluster|big \(|'aca'" gpurun_out/trace_m3_r2l.log | tail -8
HM_TRACE=1 timeout 1200 python bench.py --n 4194304 --d 3 --kernel matern --mode recompute --steps 1 --warmup 1 --cpu-baseline 0 > gpurun_out/bench_c3_r2l.json 2> gpurun_out/bench_c3_r2l.err; tail -c 400 gpurun_out/bench_c3_r2l.json; grep -E "classes|NW|smooth|cluster|big|chunk" gpurun_out/bench_c3_r2l.err | tail -10

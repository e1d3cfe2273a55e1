set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "aca or mvp_matches" > gpurun_out/pytest_r2k.log 2>&1; tail -1 gpurun_out/pytest_r2k.log
HM_SMOOTH=1 HM_SMOOTH_PRE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "aca or mvp_matches" > gpurun_out/pytest_r2k1.log 2>&1; tail -1 gpurun_out/pytest_r2k1.log
for PRE in 0 1; do
HM_SMOOTH_PRE=$PRE HM_TRACE=1 timeout 900 python tools/trace_recompute.py 1048576 4 gaussian > gpurun_out/trace_g4_r2k$PRE.log 2>&1; grep -E "smooth|mvp |\{" gpurun_out/trace_g4_r2k$PRE.log | tail -5
HM_SMOOTH_PRE=$PRE HM_TRACE=1 timeout 900 python tools/trace_recompute.py 1048576 3 matern > gpurun_out/trace_m3_r2k$PRE.log 2>&1; grep -E "smooth|mvp |\{" gpurun_out/trace_m3_r2k$PRE.log | tail -5
done
HM_TRACE=1 timeout 1200 python bench.py --n 4194304 --d 3 --kernel matern --mode recompute --steps 1 --warmup 1 --cpu-baseline 0 > gpurun_out/bench_c3_r2k.json 2> gpurun_out/bench_c3_r2k.err; tail -c 600 gpurun_out/bench_c3_r2k.json; grep -E "classes|NW|cluster|big|chunk" gpurun_out/bench_c3_r2k.err | tail -10

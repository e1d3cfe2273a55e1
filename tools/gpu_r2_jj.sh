set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_features.py -m gpu -q -x -k "kernel or entries or aca or mvp_matches or matern or k1 or C3" > gpurun_out/pytest_r2jj.log 2>&1; tail -2 gpurun_out/pytest_r2jj.log
HM_SMOOTH=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "aca or mvp_matches" > gpurun_out/pytest_r2jj1.log 2>&1; tail -2 gpurun_out/pytest_r2jj1.log
HM_TRACE=1 timeout 900 python tools/trace_recompute.py 1048576 3 matern > gpurun_out/trace_m3_r2jj.log 2>&1; grep -E "smooth|cluster|big \(|NW|'aca'" gpurun_out/trace_m3_r2jj.log | tail -8
HM_TRACE=1 timeout 900 python tools/trace_recompute.py 1048576 4 gaussian > gpurun_out/trace_g4_r2jj.log 2>&1; grep -E "smooth|cluster|big \(|NW|'aca'" gpurun_out/trace_g4_r2jj.log | tail -8

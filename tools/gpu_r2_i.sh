set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_r2i.log 2>&1; tail -2 gpurun_out/pytest_r2i.log
HM_SMOOTH=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "aca or mvp_matches or c1" > gpurun_out/pytest_r2i_s1.log 2>&1; tail -2 gpurun_out/pytest_r2i_s1.log
HM_TRACE=1 timeout 900 python tools/trace_recompute.py 1048576 4 gaussian > gpurun_out/trace_g4_r2i.log 2>&1; grep -E "NW|cluster|big \(|chunk|mvp |\{|class 0|class 1|class 2" gpurun_out/trace_g4_r2i.log | tail -14
HM_TRACE=1 timeout 900 python tools/trace_recompute.py 1048576 3 matern > gpurun_out/trace_m3_r2i.log 2>&1; grep -E "NW|cluster|big \(|mvp |\{" gpurun_out/trace_m3_r2i.log | tail -9

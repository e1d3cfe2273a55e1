set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "aca or mvp_matches" > gpurun_out/pytest_r2h.log 2>&1; tail -2 gpurun_out/pytest_r2h.log
HM_TRACE=1 timeout 900 python tools/trace_recompute.py 1048576 4 gaussian > gpurun_out/trace_g4_r2h.log 2>&1; grep -E "NW|cluster|big \(|chunk|mvp|\{" gpurun_out/trace_g4_r2h.log | tail -10
HM_TRACE=1 timeout 900 python tools/trace_recompute.py 1048576 3 matern > gpurun_out/trace_m3_r2h.log 2>&1; grep -E "NW|cluster|big \(|chunk|mvp|\{" gpurun_out/trace_m3_r2h.log | tail -10
bash tools/ncu_src_r2.sh src_m3_nw2 1048576 3 matern 'aca_win_kernel<\(int\)3, \(int\)1, \(int\)2,' 0
bash tools/ncu_src_r2.sh src_g4_nw1 262144 4 gaussian 'aca_win_kernel<\(int\)4, \(int\)0, \(int\)1,' 0
bash tools/ncu_src_r2.sh src_m3_cl4 1048576 3 matern 'aca_cluster_kernel<\(int\)3, \(int\)1, \(int\)16, \(int\)4>' 0

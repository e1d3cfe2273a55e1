set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py tests/test_gpu_round2.py -m gpu -q -x -k "not config5 and not engine" > gpurun_out/pytest_r2aa.log 2>&1; tail -2 gpurun_out/pytest_r2aa.log
HM_SMOOTH=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "aca or mvp_matches" > gpurun_out/pytest_r2aa1.log 2>&1; tail -2 gpurun_out/pytest_r2aa1.log
timeout 900 ncu -f --metrics gpu__time_duration.sum --clock-control none --csv python tools/multi_once.py 1048576 4 dmma > gpurun_out/multi_launch_dmma_r2aa.csv 2>/dev/null
python tools/launch_sum.py gpurun_out/multi_launch_dmma_r2aa.csv 4
timeout 900 python tools/setup_time.py 16777216 3 gaussian recompute 2 > gpurun_out/setup_c4_r2aa.log 2>&1; tail -1 gpurun_out/setup_c4_r2aa.log
HM_TRACE=1 timeout 900 python tools/trace_recompute.py 1048576 3 matern > gpurun_out/trace_m3_r2aa.log 2>&1; grep -E "smooth|cluster|big \(|NW|'aca'" gpurun_out/trace_m3_r2aa.log | tail -8
HM_TRACE=1 timeout 900 python tools/trace_recompute.py 1048576 4 gaussian > gpurun_out/trace_g4_r2aa.log 2>&1; grep -E "smooth|cluster|big \(|NW|'aca'" gpurun_out/trace_g4_r2aa.log | tail -8

set -x
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_round2.py -m gpu -q -x -k "not config5 and not engine" > gpurun_out/pytest_r2z.log 2>&1; tail -2 gpurun_out/pytest_r2z.log
timeout 900 ncu -f --metrics gpu__time_duration.sum --clock-control none --csv python tools/multi_once.py 1048576 4 dmma > gpurun_out/multi_launch_dmma_r2z.csv 2>/dev/null
python tools/launch_sum.py gpurun_out/multi_launch_dmma_r2z.csv 4
timeout 900 python tools/setup_time.py 16777216 3 gaussian recompute 2 > gpurun_out/setup_c4_r2z.log 2>&1; tail -1 gpurun_out/setup_c4_r2z.log

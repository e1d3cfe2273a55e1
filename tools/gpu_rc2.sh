set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_features.py tests/test_gpu_multi.py -m gpu -q -x -k "not full_size and not config5" 2>&1 | tail -3
HM_TRACE=1 timeout 900 python tools/trace_recompute.py 4194304 4 gaussian 2>&1 | grep -E "mvp|\{" | tail -3
timeout 900 python tools/trace_recompute.py 1048576 3 matern 2>&1 | tail -1

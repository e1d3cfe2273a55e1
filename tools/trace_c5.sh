set -x
timeout 900 python -m pytest tests/test_gpu_features.py tests/test_gpu_multi.py -m gpu -q -x -k "recompute or exact_multi or rank_slices" 2>&1 | tail -2
HM_TRACE=1 timeout 900 python tools/trace_recompute.py 4194304 4 gaussian 2>&1 | grep -E "classes|NW|cluster|big|chunk|mvp|\{" | tail -24

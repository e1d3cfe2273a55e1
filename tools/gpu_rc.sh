set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_features.py -m gpu -q -x -k "mvp_matches or c1_norm or rank_slices or recompute or edge or duplicate or cg" 2>&1 | tail -3
python tools/trace_recompute.py 262144 4 gaussian 2>&1 | tail -1
python tools/trace_recompute.py 1048576 3 matern 2>&1 | tail -1
HM_NO_SYM=1 python tools/trace_recompute.py 1048576 3 matern 2>&1 | tail -1

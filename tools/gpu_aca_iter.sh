# ACA iteration: parity tests + build trace at C2 + ncu of the two largest window classes
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "aca or mvp_matches or c1_norm" > gpurun_out/pytest_aca.log 2>&1; tail -3 gpurun_out/pytest_aca.log
python tools/trace_build.py 2>&1 | tail -18

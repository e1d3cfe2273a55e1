set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_features.py -m gpu -q -x -k "kernel or entries or aca or mvp_matches or matern or k1 or C3" > gpurun_out/pytest_r2ff.log 2>&1; tail -2 gpurun_out/pytest_r2ff.log
HM_TRACE=1 timeout 900 python tools/trace_recompute.py 1048576 3 matern > gpurun_out/trace_m3_r2ff.log 2>&1; grep -E "smooth|cluster|big \(|NW|'aca'" gpurun_out/trace_m3_r2ff.log | tail -8
timeout 900 python bench.py --steps 20 --warmup 3 --cpu-baseline 0 > gpurun_out/bench_c2_r2ff.json 2> gpurun_out/bench_c2_r2ff.err; tail -c 300 gpurun_out/bench_c2_r2ff.json
bash tools/ncu_src_r2.sh src_m3_scl4 1048576 3 matern 'aca_smooth_cluster_kernel<\(int\)3, \(int\)1, \(int\)4' 0

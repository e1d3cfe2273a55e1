set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_features.py -m gpu -q -x -k "kernel or entries or aca or mvp_matches or matern or k1 or C3" > gpurun_out/pytest_r2u.log 2>&1; tail -2 gpurun_out/pytest_r2u.log
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_fp64_pred_on.sum,gpu__time_duration.sum
timeout 600 ncu -f --metrics $M --clock-control none -k regex:eval_pairs --csv python tools/c_eval.py > gpurun_out/c_eval_r2u.csv 2>gpurun_out/c_eval_r2u.err
python tools/fp64_summary.py gpurun_out/c_eval_r2u.csv profiles/r2_fp64_peak_microbench.json > gpurun_out/fp64_peaks_r2u.json; grep -A7 '"c_eval"' gpurun_out/fp64_peaks_r2u.json
HM_TRACE=1 timeout 900 python tools/trace_recompute.py 1048576 3 matern > gpurun_out/trace_m3_r2u.log 2>&1; grep -E "smooth|cluster|big \(|NW|'aca'" gpurun_out/trace_m3_r2u.log | tail -8
timeout 1200 python bench.py --n 4194304 --d 3 --kernel matern --mode recompute --steps 2 --warmup 1 --cpu-baseline 0 > gpurun_out/bench_c3_r2u.json 2> gpurun_out/bench_c3_r2u.err; tail -c 300 gpurun_out/bench_c3_r2u.json

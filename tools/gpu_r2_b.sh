# Round-2 check: smoke, full GPU suite, C2 bench, C3 trace, FP64 peaks, c_eval ncu.
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2b.log 2>&1; tail -2 gpurun_out/smoke_r2b.log
./tools/fp64_peak > gpurun_out/fp64_peak_r2b.json 2>&1; cat gpurun_out/fp64_peak_r2b.json
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_fp64_pred_on.sum,gpu__time_duration.sum
timeout 600 ncu -f --metrics $M --clock-control none -k regex:eval_pairs --csv python tools/c_eval.py > gpurun_out/c_eval_r2b.csv 2>gpurun_out/c_eval_r2b.err; tail -3 gpurun_out/c_eval_r2b.csv | cut -c 1-250
python tools/fp64_summary.py gpurun_out/c_eval_r2b.csv gpurun_out/fp64_peak_r2b.json > gpurun_out/fp64_peaks_r2b.json; cat gpurun_out/fp64_peaks_r2b.json | head -30
timeout 2400 python -m pytest tests -m gpu -q -x --durations=20 > gpurun_out/pytest_gpu_r2b.log 2>&1; tail -30 gpurun_out/pytest_gpu_r2b.log
timeout 900 python bench.py --steps 20 --warmup 3 --cpu-baseline 0 > gpurun_out/bench_c2_r2b.json 2> gpurun_out/bench_c2_r2b.err; tail -c 1500 gpurun_out/bench_c2_r2b.json; tail -3 gpurun_out/bench_c2_r2b.err
HM_TRACE=1 timeout 1200 python bench.py --n 4194304 --d 3 --kernel matern --mode recompute --steps 1 --warmup 1 --cpu-baseline 0 > gpurun_out/bench_c3_r2b.json 2> gpurun_out/bench_c3_r2b.err; tail -c 1500 gpurun_out/bench_c3_r2b.json; grep -E "classes|NW|cluster|big|chunk" gpurun_out/bench_c3_r2b.err | tail -12

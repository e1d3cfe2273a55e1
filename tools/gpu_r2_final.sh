# Round-2 closing evidence: smoke, full GPU suite, C2 bench + reference arm, C3 and C5-geometry
# recompute bench lines with the reference CPU baseline, FP64-pipe metrics of the ACA kernels.
set -x
TAG=${1:-r2f}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader; nproc
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/bench_c2_$TAG.json 2> gpurun_out/bench_c2_$TAG.err; tail -c 400 gpurun_out/bench_c2_$TAG.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1; tail -c 300 gpurun_out/bench_ref_$TAG.json
timeout 1200 python bench.py --n 4194304 --d 3 --kernel matern --mode recompute --steps 3 --warmup 3 --build-reps 1 > gpurun_out/bench_c3_$TAG.json 2> gpurun_out/bench_c3_$TAG.err; tail -c 300 gpurun_out/bench_c3_$TAG.json
timeout 1200 python bench.py --n 4194304 --d 4 --mode recompute --steps 3 --warmup 3 --build-reps 1 > gpurun_out/bench_c5g_$TAG.json 2> gpurun_out/bench_c5g_$TAG.err; tail -c 300 gpurun_out/bench_c5g_$TAG.json
M=sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum
timeout 900 ncu -f --kernel-name-base demangled --metrics $M --clock-control none -k regex:'aca_|near_pair_rc' --csv python tools/one_product.py 1048576 3 matern > gpurun_out/fp64_m3_$TAG.csv 2>/dev/null
timeout 900 ncu -f --kernel-name-base demangled --metrics $M --clock-control none -k regex:'aca_|near_pair_rc' --csv python tools/one_product.py 262144 4 gaussian > gpurun_out/fp64_g4_$TAG.csv 2>/dev/null
ls -la gpurun_out/*$TAG*

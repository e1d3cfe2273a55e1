# Round-2 evidence for the C2 headline: ncu launch list of the product kernels (gpu time per
# launch, cold serialised) and a full capture of the three product kernels with DRAM bytes.
set -x
TAG=${1:-r2}
timeout 900 ncu -f --metrics gpu__time_duration.sum --clock-control none -k regex:'rows_tma|t_pair|near_pair|gather_x|scatter_z' -c 40 --csv --log-file gpurun_out/launches_c2_$TAG.csv python bench.py --steps 2 --warmup 1 --cpu-baseline 0 > /dev/null 2>&1
timeout 1500 ncu -f --set full --clock-control none --import-source on -k regex:'rows_tma|t_pair|near_pair' -s 3 -c 3 -o /tmp/prod_$TAG python bench.py --steps 2 --warmup 1 --cpu-baseline 0 > gpurun_out/ncu_prod_$TAG.log 2>&1; tail -2 gpurun_out/ncu_prod_$TAG.log
ncu -i /tmp/prod_$TAG.ncu-rep --page details --csv > gpurun_out/prod_${TAG}_details.csv 2>/dev/null
ncu -i /tmp/prod_$TAG.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/prod_${TAG}_raw.csv 2>/dev/null
M=sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum
timeout 900 ncu -f --kernel-name-base demangled --metrics $M --clock-control none -k regex:'aca_|near_pair_rc' --csv python tools/one_product.py 1048576 3 matern > gpurun_out/fp64_m3_$TAG.csv 2>/dev/null
timeout 900 ncu -f --kernel-name-base demangled --metrics $M --clock-control none -k regex:'aca_|near_pair_rc' --csv python tools/one_product.py 262144 4 gaussian > gpurun_out/fp64_g4_$TAG.csv 2>/dev/null
ls -la gpurun_out/*$TAG*

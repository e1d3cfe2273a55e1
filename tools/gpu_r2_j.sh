set -x
bash tools/ncu_src_r2.sh src_g4_sm1 262144 4 gaussian 'aca_smooth_kernel<\(int\)4, \(int\)0, \(int\)1>' 0
bash tools/ncu_src_r2.sh src_m3_sm1 1048576 3 matern 'aca_smooth_kernel<\(int\)3, \(int\)1, \(int\)1>' 0
M=sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,gpu__time_duration.sum
timeout 600 ncu -f --kernel-name-base demangled --metrics $M --clock-control none -k regex:'aca_' --csv python tools/one_product.py 1048576 3 matern > gpurun_out/aca_m3_r2j.csv 2>&1
timeout 600 ncu -f --kernel-name-base demangled --metrics $M --clock-control none -k regex:'aca_' --csv python tools/one_product.py 262144 4 gaussian > gpurun_out/aca_g4_r2j.csv 2>&1

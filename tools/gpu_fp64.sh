# FP64-pipe utilisation of the FP64-bound kernels (ACA classes at C2; recompute near field at d=4)
set -x
M=sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum,gpu__time_duration.sum
timeout 1200 ncu -f --metrics $M --clock-control none -k regex:'aca_' --csv python tools/trace_build.py > gpurun_out/fp64_aca_c2.csv 2>/dev/null; tail -3 gpurun_out/fp64_aca_c2.csv | cut -c 1-200
timeout 1200 ncu -f --metrics $M --clock-control none -k regex:'aca_|near_pair_rc|rows_kernel' --csv python tools/trace_small.py > gpurun_out/fp64_recompute_d4.csv 2>/dev/null; tail -3 gpurun_out/fp64_recompute_d4.csv | cut -c 1-200

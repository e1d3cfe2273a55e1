set -x
sed -i 's#python tools/one_product.py $N $D $K#python tools/multi_once.py $N $D dmma#' tools/ncu_src_r2.sh
bash tools/ncu_src_r2.sh src_rows_multi 1048576 4 gaussian 'rows_multi_kernel<\(int\)4, \(int\)0, \(int\)1' 0
M=sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,lts__t_bytes.sum,gpu__time_duration.sum,l1tex__t_bytes.sum
timeout 600 ncu -f --kernel-name-base demangled --metrics $M --clock-control none -k regex:'rows_multi|t_multi' -c 4 --csv python tools/multi_once.py 1048576 4 dmma > gpurun_out/multi_metrics_r2w.csv 2>/dev/null

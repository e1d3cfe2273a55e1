set -x
sed -i 's#python tools/one_product.py $N $D $K#python tools/multi_once.py $N $D dmma#' tools/ncu_src_r2.sh
bash tools/ncu_src_r2.sh src_far16 1048576 4 gaussian 'rows_multi_far16' 0
timeout 900 ncu -f --metrics gpu__time_duration.sum --clock-control none --csv python tools/multi_once.py 1048576 4 dmma > gpurun_out/multi_launch_dmma_r2y.csv 2>/dev/null
python tools/launch_sum.py gpurun_out/multi_launch_dmma_r2y.csv 4

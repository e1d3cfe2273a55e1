set -x
bash tools/ncu_src_r2.sh src_m3_nw2 1048576 3 matern 'aca_win_kernel<3, 1, 2,' 0
bash tools/ncu_src_r2.sh src_g4_nw1 262144 4 gaussian 'aca_win_kernel<4, 0, 1,' 0
bash tools/ncu_src_r2.sh src_m3_cl4 1048576 3 matern 'aca_cluster_kernel<3, 1, 16, 4>' 0

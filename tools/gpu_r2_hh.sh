set -x
timeout 1500 python bench.py --n 4194304 --d 3 --kernel matern --mode recompute --steps 2 --warmup 1 > gpurun_out/bench_c3_r2hh.json 2> gpurun_out/bench_c3_r2hh.err; tail -c 400 gpurun_out/bench_c3_r2hh.json
bash tools/ncu_src_r2.sh src_g4_snw1 1048576 4 gaussian 'aca_smooth_kernel<\(int\)4, \(int\)0, \(int\)1' 0
bash tools/ncu_src_r2.sh src_g4_snw4 1048576 4 gaussian 'aca_smooth_kernel<\(int\)4, \(int\)0, \(int\)4' 0

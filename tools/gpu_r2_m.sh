set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "mvp_matches or near" > gpurun_out/pytest_r2m.log 2>&1; tail -2 gpurun_out/pytest_r2m.log
bash tools/ncu_src_r2.sh src_m3_big 1048576 3 matern 'aca_big_kernel' 0
HM_TRACE=1 timeout 1200 python bench.py --n 4194304 --d 3 --kernel matern --mode recompute --steps 2 --warmup 1 > gpurun_out/bench_c3_r2m.json 2> gpurun_out/bench_c3_r2m.err; tail -c 2500 gpurun_out/bench_c3_r2m.json; grep -E "classes|NW|smooth|cluster|big|chunk" gpurun_out/bench_c3_r2m.err | tail -10

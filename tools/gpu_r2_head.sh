# Round-2 re-entry check of HEAD: smoke, full GPU suite, C2 bench, reference arm, config-3 and
# config-5-geometry recompute bench lines with the per-class ACA trace.
set -x
TAG=${1:-r2h}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader; nproc
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/bench_c2_$TAG.json 2> gpurun_out/bench_c2_$TAG.err; tail -c 400 gpurun_out/bench_c2_$TAG.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1; tail -c 300 gpurun_out/bench_ref_$TAG.json
HM_TRACE=1 timeout 1200 python bench.py --n 4194304 --d 3 --kernel matern --mode recompute --steps 3 --warmup 3 --build-reps 1 > gpurun_out/bench_c3_$TAG.json 2> gpurun_out/bench_c3_$TAG.err; tail -c 300 gpurun_out/bench_c3_$TAG.json
HM_TRACE=1 timeout 1200 python bench.py --n 4194304 --d 4 --mode recompute --steps 3 --warmup 3 --build-reps 1 > gpurun_out/bench_c5g_$TAG.json 2> gpurun_out/bench_c5g_$TAG.err; tail -c 300 gpurun_out/bench_c5g_$TAG.json

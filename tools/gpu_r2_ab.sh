# A/B of an ACA switch on config 3 (and config-5 geometry) with the per-class trace, after the
# ACA parity tests.  usage: VAR=HM_BIG_ONE bash tools/gpu_r2_ab.sh <tag> [extra pytest -k]
set -x
TAG=${1:-ab}
# hang guard: one small Matern d=3 product (every smooth / cluster / big class) first
timeout 240 python tools/one_product.py 1048576 3 matern > gpurun_out/guard_$TAG.log 2>&1 || { echo "guard failed"; tail -3 gpurun_out/guard_$TAG.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "aca or mvp" > gpurun_out/pytest_$TAG.log 2>&1; tail -2 gpurun_out/pytest_$TAG.log
timeout 900 python -m pytest tests/test_gpu_features.py -m gpu -q -x -k "full_size and C3" > gpurun_out/pytest_full_$TAG.log 2>&1; tail -2 gpurun_out/pytest_full_$TAG.log
for V in ${VALS:-1 0}; do
  env $VAR=$V HM_TRACE=1 timeout 900 python bench.py --n 4194304 --d 3 --kernel matern --mode recompute --steps 2 --warmup 3 --build-reps 1 --cpu-baseline 0 > gpurun_out/c3_${TAG}_$V.json 2> gpurun_out/c3_${TAG}_$V.err; tail -c 250 gpurun_out/c3_${TAG}_$V.json
  env $VAR=$V HM_TRACE=1 timeout 900 python bench.py --n 4194304 --d 4 --mode recompute --steps 2 --warmup 3 --build-reps 1 --cpu-baseline 0 > gpurun_out/c5g_${TAG}_$V.json 2> gpurun_out/c5g_${TAG}_$V.err; tail -c 250 gpurun_out/c5g_${TAG}_$V.json
done

# A/B of a product-level switch (no trace: the trace serialises the streams) on config 3 and
# the config-5 geometry, after the tests named by PYK.  usage: VAR=HM_OVERLAP PYK="..." bash tools/gpu_r2_ab2.sh <tag>
set -x
TAG=${1:-ab}
timeout 1200 python -m pytest tests -m gpu -q -x -k "${PYK:-overlap}" > gpurun_out/pytest_$TAG.log 2>&1; tail -2 gpurun_out/pytest_$TAG.log
for V in ${VALS:-1 0}; do
  env $VAR=$V timeout 900 python bench.py --n 4194304 --d 3 --kernel matern --mode recompute --steps 2 --warmup 3 --build-reps 1 --cpu-baseline 0 > gpurun_out/c3_${TAG}_$V.json 2> gpurun_out/c3_${TAG}_$V.err; tail -c 250 gpurun_out/c3_${TAG}_$V.json
  env $VAR=$V timeout 900 python bench.py --n 4194304 --d 4 --mode recompute --steps 2 --warmup 3 --build-reps 1 --cpu-baseline 0 > gpurun_out/c5g_${TAG}_$V.json 2> gpurun_out/c5g_${TAG}_$V.err; tail -c 250 gpurun_out/c5g_${TAG}_$V.json
done

# ncu captures of the product kernels at N=2^18 (same kernels, smaller operator)
set -x
N=${1:-262144}
KREGEX=${2:-rows_tma|lowrank_t}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KREGEX" -s 3 -c 3 -o gpurun_out/prof python bench.py --n $N --steps 2 --warmup 1 --cpu-baseline 0 > gpurun_out/ncu.log 2>&1; tail -3 gpurun_out/ncu.log

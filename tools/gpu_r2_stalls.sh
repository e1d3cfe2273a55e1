# Warp-stall breakdown (pc sampling) and FP64-pipe use of the Matern d=3 ACA kernels, plus the
# per-line source pages of the big-block and smooth cluster kernels.  usage: bash tools/gpu_r2_stalls.sh [tag]
set -x
TAG=${1:-st}
N=${N:-1048576}
timeout 1200 ncu -f --kernel-name-base demangled --set full --clock-control none --import-source on \
  -k regex:'aca_(big|smooth|win)' -c 12 -o /tmp/aca_$TAG python tools/one_product.py $N 3 matern > gpurun_out/aca_$TAG.log 2>&1; tail -2 gpurun_out/aca_$TAG.log
ncu -i /tmp/aca_$TAG.ncu-rep --page raw --csv > gpurun_out/aca_${TAG}_raw.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/aca_${TAG}_raw.csv > gpurun_out/aca_${TAG}_stalls.txt; cat gpurun_out/aca_${TAG}_stalls.txt
for K in aca_big_kernel aca_smooth_cluster_kernel; do
  ncu -i /tmp/aca_$TAG.ncu-rep -k regex:$K --page source --csv --print-source cuda > gpurun_out/aca_${TAG}_${K}_cuda.csv 2>/dev/null
  ncu -i /tmp/aca_$TAG.ncu-rep -k regex:$K --page source --csv --print-source sass > gpurun_out/aca_${TAG}_${K}_sass.csv 2>/dev/null
done
ls -la gpurun_out/aca_${TAG}*

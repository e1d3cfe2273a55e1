# ncu --set full of ACA kernels in recompute mode, exported to CSV on the box.
# usage: bash tools/ncu_aca_r2.sh <tag> <N> <d> <kernel> <regex> <skip> <count>
set -x
TAG=$1; N=$2; D=$3; K=$4; RE=$5; S=$6; C=$7
timeout 1500 ncu -f --set full --clock-control none --import-source on -k regex:"$RE" -s $S -c $C -o /tmp/$TAG python tools/one_product.py $N $D $K > gpurun_out/$TAG.log 2>&1; tail -3 gpurun_out/$TAG.log
ncu -i /tmp/$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
ncu -i /tmp/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i /tmp/$TAG.ncu-rep --page source --csv --print-source cuda > gpurun_out/${TAG}_src.csv 2>/dev/null
ls -la gpurun_out/${TAG}*

# ncu capture + CUDA-source-level export (line-attributed instruction counts)
set -x
NAME=$1; RE=$2; S=$3; C=$4; shift 4
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:"$RE" -s $S -c $C -o /tmp/$NAME "$@" > gpurun_out/$NAME.log 2>&1
ncu -i /tmp/$NAME.ncu-rep --page source --csv --print-source cuda > gpurun_out/${NAME}_cuda.csv 2>gpurun_out/${NAME}_cuda.err
ncu -i /tmp/$NAME.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${NAME}_mixed.csv 2>>gpurun_out/${NAME}_cuda.err
ls -la gpurun_out/${NAME}*; head -c 600 gpurun_out/${NAME}_cuda.csv

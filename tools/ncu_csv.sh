# ncu capture on the box, exported to CSV there (the .ncu-rep can exceed the 64 MiB copy-back)
# usage: bash tools/ncu_csv.sh <name> <kernel-regex> <skip> <count> <command...>
set -x
NAME=$1; RE=$2; S=$3; C=$4; shift 4
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:"$RE" -s $S -c $C -o /tmp/$NAME "$@" > gpurun_out/$NAME.log 2>&1; tail -2 gpurun_out/$NAME.log
ncu -i /tmp/$NAME.ncu-rep --page details --csv > gpurun_out/${NAME}_details.csv 2>/dev/null
ncu -i /tmp/$NAME.ncu-rep --page source --csv --print-source sass > gpurun_out/${NAME}_sass.csv 2>/dev/null
ls -la gpurun_out/${NAME}*

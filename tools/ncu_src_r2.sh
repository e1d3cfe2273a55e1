# per-instruction / per-source-line hot spots of one ACA kernel (SASS + CUDA source pages)
# usage: bash tools/ncu_src_r2.sh <tag> <N> <d> <kernel> <regex> <skip>
set -x
TAG=$1; N=$2; D=$3; K=$4; RE=$5; S=$6
timeout 900 ncu -f --kernel-name-base demangled --section SourceCounters --section WarpStateStats --section InstructionStats --clock-control none --import-source on -k regex:"$RE" -s $S -c 1 -o /tmp/$TAG python tools/one_product.py $N $D $K > gpurun_out/$TAG.log 2>&1; tail -2 gpurun_out/$TAG.log
ncu -i /tmp/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>gpurun_out/${TAG}_sass.err
ncu -i /tmp/$TAG.ncu-rep --page source --csv --print-source cuda > gpurun_out/${TAG}_cuda.csv 2>>gpurun_out/${TAG}_sass.err
ncu -i /tmp/$TAG.ncu-rep --page raw --csv --print-metric-instances values --metrics sass__inst_executed_per_opcode > gpurun_out/${TAG}_opcodes.csv 2>>gpurun_out/${TAG}_sass.err
ls -la gpurun_out/${TAG}*; head -c 800 gpurun_out/${TAG}_cuda.csv

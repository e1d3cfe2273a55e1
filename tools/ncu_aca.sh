# ncu --set full of the ACA team kernels at N=2^18 (d=2): skip S launches, capture C
set -x
S=${1:-3}; C=${2:-1}; N=${3:-262144}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'aca_team|aca_kernel' -s $S -c $C -o gpurun_out/prof_aca python tools/trace_build.py $N > gpurun_out/ncu_aca.log 2>&1; tail -5 gpurun_out/ncu_aca.log
ls -la gpurun_out

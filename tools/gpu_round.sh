# GPU round: tests, bench (C2), launch list, ncu captures.  Usage: bash tools/gpu_round.sh [quick|full|ncu]
set -x
MODE=${1:-full}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
if [ "$MODE" != "ncu" ]; then
  timeout 900 python bench.py --steps 30 --warmup 3 --cpu-baseline $([ "$MODE" = full ] && echo 1 || echo 0) > gpurun_out/bench.json 2> gpurun_out/bench.err
  tail -c 4000 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
fi
if [ "$MODE" != "quick" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'rows_kernel|lowrank|gather|scatter' -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 1 --cpu-baseline 0 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'rows_kernel' -s 1 -c 1 -o gpurun_out/prof_rows python bench.py --n 262144 --steps 2 --warmup 1 --cpu-baseline 0 > gpurun_out/ncu_rows.log 2>&1; tail -3 gpurun_out/ncu_rows.log
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'lowrank_t' -s 2 -c 2 -o gpurun_out/prof_t python bench.py --n 262144 --steps 2 --warmup 1 --cpu-baseline 0 > gpurun_out/ncu_t.log 2>&1; tail -3 gpurun_out/ncu_t.log
fi
ls -la gpurun_out

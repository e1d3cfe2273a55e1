# Full GPU round: smoke, GPU suite, C2 bench (+CPU baseline), reference arm, ncu launch list and
# full captures of the product kernels (exported to CSV on the box).  Usage: bash tools/gpu_round.sh [tag]
set -x
TAG=${1:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader; nproc; free -g | head -2; lscpu | grep "Model name"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/bench_c2_$TAG.json 2> gpurun_out/bench_c2_$TAG.err; tail -c 600 gpurun_out/bench_c2_$TAG.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>&1; tail -c 300 gpurun_out/bench_ref_$TAG.json
timeout 900 ncu -f --metrics gpu__time_duration.sum --clock-control none -k regex:'rows_tma|t_pair|near_pair|gather_x|scatter_z' -c 40 --csv --log-file gpurun_out/launches_c2_$TAG.csv python bench.py --steps 2 --warmup 1 --cpu-baseline 0 > /dev/null 2>&1
timeout 1500 ncu -f --set full --clock-control none --import-source on -k regex:'rows_tma|t_pair|near_pair' -s 3 -c 3 -o /tmp/prod_$TAG python bench.py --steps 2 --warmup 1 --cpu-baseline 0 > gpurun_out/ncu_prod_$TAG.log 2>&1; tail -2 gpurun_out/ncu_prod_$TAG.log
ncu -i /tmp/prod_$TAG.ncu-rep --page details --csv > gpurun_out/prod_${TAG}_details.csv 2>/dev/null
ncu -i /tmp/prod_$TAG.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/prod_${TAG}_raw.csv 2>/dev/null
ls -la gpurun_out | tail -20

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
lscpu | grep -E "Model name|^CPU\(s\)"; free -g | head -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q 2>&1 | tail -15
timeout 300 python bench.py --n 65536 --steps 20 --warmup 3 --cpu-baseline 0 2>&1 | tail -3
timeout 900 python bench.py --steps 30 --warmup 3 --cpu-baseline 0 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -c 3000 gpurun_out/bench_c2.json; tail -5 gpurun_out/bench_c2.err

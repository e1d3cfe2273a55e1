set -x
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -k "not config5" > gpurun_out/pytest_r2v.log 2>&1; tail -2 gpurun_out/pytest_r2v.log
timeout 900 ncu -f --metrics gpu__time_duration.sum --clock-control none --csv python tools/multi_once.py 1048576 4 dmma > gpurun_out/multi_launch_dmma_r2v.csv 2>/dev/null
python tools/launch_sum.py gpurun_out/multi_launch_dmma_r2v.csv 6
timeout 600 python tools/bench_multi.py --n 1048576 --d 4 --mode recompute --nrhs 16 --steps 2 > gpurun_out/multi_2e20_r2v.jsonl 2>&1; tail -2 gpurun_out/multi_2e20_r2v.jsonl | cut -c 1-300

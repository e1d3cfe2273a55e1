set -x
timeout 600 python tools/bench_multi.py --n 1048576 --d 2 --mode stored --nrhs 16 --steps 5 > gpurun_out/multi_c2.jsonl 2>&1; cat gpurun_out/multi_c2.jsonl | tail -3
timeout 900 python tools/bench_multi.py --n 262144 --d 4 --mode recompute --nrhs 16 --steps 2 > gpurun_out/multi_c5s.jsonl 2>&1; cat gpurun_out/multi_c5s.jsonl | tail -3

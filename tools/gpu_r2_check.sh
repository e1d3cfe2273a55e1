# Final HEAD check: hang guard, smoke, full GPU suite, default bench line.
set -x
TAG=${1:-chk}
timeout 240 python tools/one_product.py 1048576 3 matern > gpurun_out/guard_$TAG.log 2>&1 || { echo "guard failed"; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_c2_$TAG.json 2> gpurun_out/bench_c2_$TAG.err; tail -c 400 gpurun_out/bench_c2_$TAG.json

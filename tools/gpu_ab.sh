# A/B of product variants at C2 (bench ms/step and per-kernel times)
set -x
timeout 600 python -m pytest tests -m gpu -q -x -k "mvp_matches or c1_norm or bench_config or rank_slices" 2>&1 | tail -2
for v in "X=1" "X=2"; do
  echo "== $v"; env $v timeout 600 python bench.py --steps 20 --warmup 3 --cpu-baseline 0 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['e2e']['value'], {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})"
done

set -x
for v in "X=1" "HM_NW8V=1"; do echo "== $v"; env $v HM_TRACE=1 timeout 300 python tools/trace_build.py 2>&1 | grep -E "NW=8" | tail -1; env $v HM_TRACE=1 timeout 300 python tools/trace_small.py 2>&1 | grep -E "NW=8" | tail -1; done

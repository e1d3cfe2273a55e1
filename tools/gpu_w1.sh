set -x
for v in "X=1" "HM_W1OLD=1"; do echo "== $v"; env $v HM_TRACE=1 timeout 300 python tools/trace_build.py 2>&1 | grep -E "NW=1|NW=2|setup" | tail -3; env $v HM_TRACE=1 timeout 300 python tools/trace_small.py 2>&1 | grep -E "NW=1|NW=2" | tail -2; done

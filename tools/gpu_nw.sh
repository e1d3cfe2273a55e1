set -x
for v in "X=1" "HM_NW2=2 HM_NW4=2" "HM_NW2=4 HM_NW4=w"; do echo "== $v"; env $v HM_TRACE=1 timeout 300 python tools/trace_build.py 2>&1 | grep -E "NW=2|NW=4" | tail -2; env $v HM_TRACE=1 timeout 300 python tools/trace_small.py 2>&1 | grep -E "NW=2|NW=4" | tail -2; done

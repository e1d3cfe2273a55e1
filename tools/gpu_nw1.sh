set -x
for v in 4 3 2; do echo "== HM_NW1=$v"; HM_NW1=$v HM_TRACE=1 timeout 300 python tools/trace_build.py 2>&1 | grep -E "NW=1" | tail -1; HM_NW1=$v HM_TRACE=1 timeout 300 python tools/trace_small.py 2>&1 | grep -E "NW=1" | tail -1; done

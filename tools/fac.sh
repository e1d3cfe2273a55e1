set -x
g++ -std=c++20 -O2 -I include tests/cpp/facade_demo.cpp -o /tmp/facade_demo -L paper_1708_09707_b200 -lhmat_b200 -Wl,-rpath,$PWD/paper_1708_09707_b200
for i in 1 2 3; do /tmp/facade_demo; echo rc=$?; done
timeout 300 compute-sanitizer --print-limit 3 /tmp/facade_demo 2>&1 | tail -20
CUDA_LAUNCH_BLOCKING=1 /tmp/facade_demo; echo rc=$?

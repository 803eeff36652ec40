#!/bin/bash
# Exchange-mode sweep: tests/cpp/dist_threads (world ranks as threads of one
# process, caller collectives through blfmm_comm_ops) over dimensions, node
# counts (M = 16, other even M <= 64, odd M), kernels, right-hand sides and
# world sizes; each run compares the distributed matvec with the one-rank
# matvec of the same library (rel-l2 <= 1e-13 inside the program).
root=$(cd "$(dirname "$0")/.." && pwd)
exe=/tmp/dist_threads_fuzz
g++ -std=c++20 -O2 -I$root/include -I/usr/local/cuda/include $root/tests/cpp/dist_threads.cpp -o $exe \
  -L$root/paper_1606_07652_b200 -lblfmm_gpu -L/usr/local/cuda/lib64 -lcudart \
  -Wl,-rpath,$root/paper_1606_07652_b200 -pthread || exit 1
fails=0
run() { out=$($exe "$@" 2>&1); rc=$?; if [ $rc -ne 0 ] || ! echo "$out" | grep -q OK; then echo "FAIL $* :: $(echo $out | tail -c 300)"; fails=$((fails+1)); else echo "ok   $* :: $(echo "$out" | grep rel-l2)"; fi; }
PI=3.141592653589793
run 3 20000 3 2 imq:c=0.1 $PI 20 1
run 3 20000 3 3 gaussian:c=64 $PI 34 1
run 3 8000 2 2 mq:c=0.2 $PI 58 1
run 3 20000 3 4 imq:c=0.1 $PI 15 1
run 3 20000 3 2 imq:c=0.1 $PI 24 2
run 3 30000 4 3 gaussian:c=64 $PI 16 8
run 3 30000 3 2 gaussian:c=64 $PI 16 32
run 3 3000 4 5 imq:c=0.1 $PI 16 1
run 2 30000 5 3 imq:c=0.3 $PI 16 1
run 2 30000 4 2 mq:c=0.05 $PI 20 2
run 2 30000 5 4 gaussian:c=16 $PI 33 1
run 2 500 6 3 mq:c=0.05 $PI 16 1
run 1 5000 6 3 imq:c=1 $PI 64 1
run 1 5000 4 2 gaussian:c=9 $PI 300 2
run 1 40 5 4 mq:c=0.2 $PI 8 1
echo "$fails failures"
exit $fails

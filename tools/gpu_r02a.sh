#!/bin/bash
# round-2 first GPU pass: tests, per-workload step times, bench (P3), ncu metric names
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu >> gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
for wl in P3 P4 P5 P2p P2 P1; do timeout 300 python tools/time_step.py --workload $wl --steps 10 >> gpurun_out/steps.txt 2>&1; done
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo done > gpurun_out/done.txt

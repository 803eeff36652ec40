#!/bin/bash
# One GPU evidence pass: gpu tests, smoke, bench (P3), per-workload step times.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
for wl in P1 P2p P4 P5 P2; do timeout 300 python tools/time_step.py --workload $wl --steps 5 >> gpurun_out/steps.txt 2>&1; done

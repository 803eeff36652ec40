mkdir -p gpurun_out
for wl in P5; do timeout 300 python tools/time_step.py --workload $wl --steps 5 >> gpurun_out/steps.txt 2>&1; done
timeout 1500 python -m pytest tests -m gpu -x -q -k "batched or P5 or p5 or rhs or distributed or nccl" > gpurun_out/pytest_sub.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_sub.txt

python tools/time_step.py --steps 20 --tag pruned > gpurun_out/log.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -2 >> gpurun_out/log.txt

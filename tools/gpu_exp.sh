python tools/run_steps.py --steps 2 2>&1 | tail -1 > gpurun_out/log.txt 2>&1; python tools/time_step.py --steps 20 --tag c32 >> gpurun_out/log.txt 2>&1

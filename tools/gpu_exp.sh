python tools/time_step.py --steps 20 --tag n1 > gpurun_out/log.txt 2>&1
timeout 1500 python tools/shard_time.py --worlds 8 >> gpurun_out/log.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -2 >> gpurun_out/log.txt

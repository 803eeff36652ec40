mkdir -p gpurun_out
timeout 900 python tools/ab_couple.py 0 1 2 6 > gpurun_out/ab_couple.txt 2>&1

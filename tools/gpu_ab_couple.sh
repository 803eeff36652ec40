python tools/ab_couple.py "$@" 2>&1 | tee gpurun_out/ab_couple.txt

for b in 3 4; do BLFMM_COUPLE_MINB=$b python tools/run_steps.py --scaled 10 --steps 2 2>&1 | tail -1 | sed "s/^/minb$b /"; done > gpurun_out/log.txt 2>&1

for b in 2 3 4 5; do BLFMM_COUPLE_MINB=$b python tools/run_steps.py --steps 3 2>&1 | tail -1 | sed "s/^/minb$b /"; done

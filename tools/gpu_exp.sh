for v in 1 5; do BLFMM_COUPLE_VARIANT=$v python tools/run_steps.py --steps 3 2>&1 | tail -1 | sed "s/^/v$v /"; done

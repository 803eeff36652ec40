for v in 1 2 3 4; do BLFMM_COUPLE_VARIANT=$v python tools/run_steps.py --steps 2 2>&1 | tail -1 | sed "s/^/v$v /"; done > gpurun_out/log.txt 2>&1
BLFMM_COUPLE_VARIANT=3 timeout 900 python -m pytest tests -m gpu -x -q -k "P3 or stage or golden or exchange" 2>&1 | tail -2 >> gpurun_out/log.txt

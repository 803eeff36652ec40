for v in "1 4" "6 3" "6 4" "6 5"; do set -- $v; BLFMM_COUPLE_VARIANT=$1 BLFMM_COUPLE_MINB=$2 python tools/run_steps.py --steps 2 2>&1 | tail -1 | sed "s/^/v$1 minb$2 /"; done > gpurun_out/log.txt 2>&1
BLFMM_COUPLE_VARIANT=6 timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 >> gpurun_out/log.txt

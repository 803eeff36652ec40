for v in 64 96 128; do BLFMM_NEAR_ITEM=$v python tools/run_steps.py --steps 3 2>&1 | tail -1 | sed "s/^/item$v /"; done
for v in 64 96 128; do BLFMM_NEAR_ITEM=$v timeout 900 python -m pytest tests -m gpu -x -q -k "P3 or P2 or near or sharded" 2>&1 | tail -1; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2

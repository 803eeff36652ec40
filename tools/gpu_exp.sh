for f in 0 1; do BLFMM_FUSE_NEAR_M2M=$f python tools/time_step.py --tag fuse$f 2>&1 | tail -1; done

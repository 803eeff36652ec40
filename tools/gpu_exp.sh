(timeout 600 oracle/_ref/test_fmm_gpu | tail -3; timeout 900 oracle/_ref/test_mlfmm_gpu | tail -1) > gpurun_out/dropin.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 >> gpurun_out/dropin.txt

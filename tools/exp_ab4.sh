mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "near or split or stats or graph" > gpurun_out/pytest4.txt 2>&1; echo "exit $?" >> gpurun_out/pytest4.txt
for cfg in "BLFMM_NEAR_STAGE=0" "BLFMM_NEAR_STAGE=1" "BLFMM_NEAR_STAGE=1 BLFMM_NEAR_PERSIST=2" "BLFMM_NEAR_STAGE=1 BLFMM_NEAR_PERSIST=4" "BLFMM_NEAR_STAGE=1 BLFMM_SYM_SPLIT=1" "BLFMM_NEAR_STAGE=0"; do
  env $cfg python tools/time_step.py --workload P3 --steps 20 --tag "[$cfg]" 2>&1 | tail -1 >> gpurun_out/ab4.txt
done
BLFMM_NEAR_STAGE=0 python tools/run_steps.py --steps 2 > gpurun_out/rs4.txt 2>&1
BLFMM_NEAR_STAGE=1 python tools/run_steps.py --steps 2 >> gpurun_out/rs4.txt 2>&1
BLFMM_NEAR_STAGE=1 BLFMM_SYM_SPLIT=1 python tools/run_steps.py --steps 2 >> gpurun_out/rs4.txt 2>&1

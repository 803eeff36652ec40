mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest3.txt 2>&1; echo "exit $?" >> gpurun_out/pytest3.txt
for cfg in "BLFMM_SYM_SPLIT=0" "BLFMM_SYM_SPLIT=1" "BLFMM_SYM_SPLIT=0 BLFMM_NEAR_PERSIST=4" "BLFMM_SYM_SPLIT=1 BLFMM_NEAR_PERSIST=4" "BLFMM_SYM_SPLIT=0 BLFMM_NEAR_PERSIST=2"; do
  env $cfg python tools/time_step.py --workload P3 --steps 20 --tag "[$cfg]" 2>&1 | tail -1 >> gpurun_out/ab3.txt
done
timeout 900 python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err

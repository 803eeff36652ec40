mkdir -p gpurun_out
for cfg in "BLFMM_NEAR_PERSIST=3" "BLFMM_NEAR_PERSIST=2" "BLFMM_NEAR_PERSIST=4" "BLFMM_NEAR_PERSIST=5" "BLFMM_NEAR_PERSIST=3 BLFMM_COUPLE_SKIP=1"; do
  env $cfg python tools/time_step.py --workload P3 --steps 20 --tag "[$cfg]" 2>&1 | tail -1 >> gpurun_out/ab1.txt
done
python tools/time_step.py --workload P3 --steps 2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_near_all -c 1 -o gpurun_out/near_p3 python tools/time_step.py --workload P3 --steps 2 > gpurun_out/ncu_near3.log 2>&1
BLFMM_NEAR_PERSIST=5 ncu --set full --clock-control none --import-source on -k regex:k_near_all -c 1 -o gpurun_out/near_p5 python tools/time_step.py --workload P3 --steps 2 > gpurun_out/ncu_near5.log 2>&1

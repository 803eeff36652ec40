mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest2.txt 2>&1; echo "exit $?" >> gpurun_out/pytest2.txt
for cfg in "BLFMM_SYM_SPLIT=0" "BLFMM_SYM_SPLIT=1" "BLFMM_NEAR_PERSIST=5" "BLFMM_NEAR_PERSIST=4" "BLFMM_TELE_VARIANT=8" "BLFMM_TELE_VARIANT=9" "BLFMM_TELE_VARIANT=8 BLFMM_NEAR_PERSIST=5" "BLFMM_SYM_SPLIT=0 BLFMM_NEAR_PERSIST=5"; do
  env $cfg python tools/time_step.py --workload P3 --steps 20 --tag "[$cfg]" 2>&1 | tail -1 >> gpurun_out/ab2.txt
done
python tools/run_steps.py --steps 2 > gpurun_out/rs2.txt 2>&1
BLFMM_NEAR_PERSIST=5 ncu --metrics gpu__time_duration.sum,sm__cycles_active.max,sm__cycles_active.avg --clock-control none -k regex:"k_near_all|k_couple3|k_sym_fix" --csv --log-file gpurun_out/ncu_ab2.csv python tools/time_step.py --workload P3 --steps 2 > /dev/null 2>&1
BLFMM_TELE_VARIANT=8 ncu --metrics gpu__time_duration.sum,sm__cycles_active.max,sm__cycles_active.avg --clock-control none -k regex:"k_couple3" -c 3 --csv --log-file gpurun_out/ncu_ab2b.csv python tools/time_step.py --workload P3 --steps 2 > /dev/null 2>&1

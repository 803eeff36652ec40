mkdir -p gpurun_out
for wl in P4 P1 P3; do timeout 300 python tools/time_step.py --workload $wl --steps 10 >> gpurun_out/steps.txt 2>&1; done
timeout 1200 python -m pytest tests -x -q -m gpu -k "P4 or p4 or 2d or golden or mlfmm_matches or stage_exp or sharded or exchange or edge or unit_source or couple_scalar or cpp or reference_unit" > gpurun_out/pytest_sub.txt 2>&1

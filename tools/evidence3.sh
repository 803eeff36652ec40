#!/bin/bash
# Round-2 closing evidence pass (run under gpurun): tools/evidence.sh, then
# --set full captures of the P2 (3M large-M kernels) and P4 (2-D generated
# phase kernels) workloads. Each ncu command runs after the same command
# exited 0 without ncu.
bash tools/evidence.sh
python tools/run_steps.py --workload P2 --steps 1 > gpurun_out/plain_p2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_p2m_big3|k_l2p_half_a3|k_p2m_axes|k_l2p_axes" -c 7 \
      -o gpurun_out/prof_p2 python tools/run_steps.py --workload P2 --steps 1 > gpurun_out/ncu_p2.log 2>&1
python tools/run_steps.py --workload P4 --steps 1 > gpurun_out/plain_p4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_p2m_2d16|k_l2p_2d16|k_near_all" -c 3 \
      -o gpurun_out/prof_p4 python tools/run_steps.py --workload P4 --steps 1 > gpurun_out/ncu_p4.log 2>&1
echo done > gpurun_out/evidence3_done.txt

#!/bin/bash
# Second evidence pass: executed-FP64 metrics of one P3 matvec without the
# stats GEMM (the bench's timed call), and --set full captures of the P5
# (32 right-hand sides) and P4 kernels.
mkdir -p gpurun_out
python tools/run_steps.py --steps 1 > gpurun_out/plain1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active \
      --clock-control none -k regex:k_ --csv --log-file gpurun_out/step_metrics.csv python tools/run_steps.py --steps 1 > gpurun_out/ncu1.log 2>&1
python tools/run_steps.py --workload P5 --steps 1 > gpurun_out/plain5.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_p2m_mr|k_l2p_mr|k_near_dmma" -c 3 \
      -o gpurun_out/prof_p5 python tools/run_steps.py --workload P5 --steps 1 > gpurun_out/ncu5.log 2>&1
python tools/run_steps.py --workload P4 --steps 1 > gpurun_out/plain4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_p2m_2d16|k_l2p_2d16|k_near_all" -c 3 \
      -o gpurun_out/prof_p4 python tools/run_steps.py --workload P4 --steps 1 > gpurun_out/ncu4.log 2>&1
echo done > gpurun_out/evidence2_done.txt

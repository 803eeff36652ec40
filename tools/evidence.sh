#!/bin/bash
# One GPU evidence pass (run under gpurun): GPU tests, smoke, bench (P3, the
# driver's command line) and the reference arm, per-workload step times, the
# ncu launch list of the bench command, per-kernel DRAM bytes and executed
# FP64 work of one matvec, and a --set full capture of the top kernels. Each
# ncu command runs right after the same command exited 0.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=20 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
for wl in P1 P2p P4 P5 P2; do timeout 300 python tools/time_step.py --workload $wl --steps 5 >> gpurun_out/steps.txt 2>&1; done
python tools/run_steps.py --steps 1 > gpurun_out/plain1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active \
      --clock-control none -k regex:k_ --csv --log-file gpurun_out/step_metrics.csv python tools/run_steps.py --steps 1 > gpurun_out/ncu1.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra-workloads > gpurun_out/plain2.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra-workloads > gpurun_out/ncu2.log 2>&1
python tools/time_step.py --workload P3 --steps 2 > gpurun_out/plain3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on \
      -k regex:"k_couple_col|k_near_all|k_l2p_h16S|k_p2m_m2m" -c 4 -o gpurun_out/prof_full \
      python tools/time_step.py --workload P3 --steps 2 > gpurun_out/ncu3.log 2>&1
timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo done > gpurun_out/evidence_done.txt

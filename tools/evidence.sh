#!/bin/bash
# One GPU evidence pass (run under gpurun): GPU tests, smoke, bench (P3, the
# driver's command line), per-workload step times, the ncu launch list of the
# bench command, per-kernel DRAM bytes and executed FP64 work of one matvec, and
# --set full captures of the top kernels of P3 / P2 / P4 / P5. Each ncu command
# runs right after the same command exited 0. The .ncu-rep files are exported
# to CSV on the box and deleted (gpurun merges at most 64 MiB back).
# usage: evidence.sh [tests|bench|ncu|ref] ...   (default: all four parts)
mkdir -p gpurun_out
parts="${*:-tests bench ncu ref}"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
export_rep() {  # $1 = report stem: raw + source pages to CSV, then drop the report
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page source --csv > gpurun_out/$1_source.csv 2>/dev/null
  python tools/ncu_source_summary.py gpurun_out/$1_raw.csv gpurun_out/$1_source.csv > gpurun_out/$1_summary.txt 2>&1
  rm -f gpurun_out/$1.ncu-rep gpurun_out/$1_source.csv
}
for part in $parts; do
case $part in
tests)
  timeout 1500 python -m pytest tests -m gpu -x -q --durations=20 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
  ;;
bench)
  timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
  rm -f gpurun_out/steps.txt
  for wl in P1 P2p P4 P5 P2; do timeout 300 python tools/time_step.py --workload $wl --steps 5 >> gpurun_out/steps.txt 2>&1; done
  ;;
ncu)
  python tools/run_steps.py --steps 1 > gpurun_out/plain1.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active \
        --clock-control none -k regex:k_ --csv --log-file gpurun_out/step_metrics.csv python tools/run_steps.py --steps 1 > gpurun_out/ncu1.log 2>&1
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra-workloads > gpurun_out/plain2.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
        python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra-workloads > gpurun_out/ncu2.log 2>&1
  python tools/time_step.py --workload P3 --steps 2 > gpurun_out/plain3.log 2>&1 && \
    ncu --set full --clock-control none --import-source on \
        -k regex:"k_couple_col|k_near_all|k_l2p_h16S|k_p2m_m2m" -c 4 -o gpurun_out/prof_p3 \
        python tools/time_step.py --workload P3 --steps 2 > gpurun_out/ncu3.log 2>&1 && export_rep prof_p3
  python tools/run_steps.py --workload P2 --steps 1 > gpurun_out/plain_p2.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:"k_p2m_big3|k_l2p_half_a3|k_p2m_axes|k_l2p_axes" -c 6 \
        -o gpurun_out/prof_p2 python tools/run_steps.py --workload P2 --steps 1 > gpurun_out/ncu_p2.log 2>&1 && export_rep prof_p2
  python tools/run_steps.py --workload P4 --steps 1 > gpurun_out/plain_p4.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:"k_p2m_2d16|k_l2p_2d16|k_near_all" -c 3 \
        -o gpurun_out/prof_p4 python tools/run_steps.py --workload P4 --steps 1 > gpurun_out/ncu_p4.log 2>&1 && export_rep prof_p4
  python tools/run_steps.py --workload P5 --steps 1 > gpurun_out/plain_p5.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:"k_p2m_mr|k_l2p_mr|k_near_dmma" -c 3 \
        -o gpurun_out/prof_p5 python tools/run_steps.py --workload P5 --steps 1 > gpurun_out/ncu_p5.log 2>&1 && export_rep prof_p5
  ;;
ref)
  timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
  ;;
esac
done
echo "$parts" > gpurun_out/evidence_done.txt

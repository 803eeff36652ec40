python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 1500 gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/step_dram.csv python tools/run_steps.py --steps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_l2p_h16S -c 1 -o gpurun_out/l2pS python tools/run_steps.py --steps 1 > /dev/null 2>&1
ls gpurun_out

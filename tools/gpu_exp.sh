set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 600 gpurun_out/bench.json
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 600 gpurun_out/bench_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/step_dram.csv python tools/run_steps.py --steps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_couple3 --launch-skip 5 -c 1 -o gpurun_out/couple3_leaf python tools/run_steps.py --steps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_near_warp2 -c 1 -o gpurun_out/near2 python tools/run_steps.py --steps 1 > /dev/null 2>&1
ls gpurun_out

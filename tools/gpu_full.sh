# full GPU pass: tests, per-workload step times, bench, then an ncu capture of the couple
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
for wl in P3 P4 P5 P2p P2 P1; do timeout 300 python tools/time_step.py --workload $wl --steps 10 >> gpurun_out/steps.txt 2>&1; done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
python tools/prof_couple.py 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_couple -c 1 -o gpurun_out/prof_col python tools/prof_couple.py 1 > gpurun_out/ncu.log 2>&1

mkdir -p gpurun_out
python tools/prof_couple.py 0 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_couple -c 2 -o gpurun_out/prof_couple python tools/prof_couple.py 0 1 > gpurun_out/ncu.log 2>&1

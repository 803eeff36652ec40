#!/bin/bash
# One compute-sanitizer tool per call (B200_PROFILING.md): bash tools/sanitize.sh memcheck|racecheck|synccheck
tool=${1:-memcheck}
mkdir -p gpurun_out
python tools/sanitize_case.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
    python tools/sanitize_case.py > gpurun_out/sanitize_$tool.log 2>&1
echo "exit $?" >> gpurun_out/sanitize_$tool.log

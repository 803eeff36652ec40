#!/bin/bash
# A/B timing of env knobs on P3 + the GPU parity suite. Usage: tools/ab.sh "ENV=.. ENV=.." ...
mkdir -p gpurun_out
for cfg in "$@"; do
  env $cfg python tools/time_step.py --workload P3 --steps 20 --tag "[$cfg]" 2>&1 | tail -1 >> gpurun_out/ab.txt
done

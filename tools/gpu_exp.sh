timeout 900 python -m pytest tests -m gpu -x -q -k "graph_replay" 2>&1 | tail -3 > gpurun_out/log.txt

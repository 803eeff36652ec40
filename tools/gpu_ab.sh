mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_multigpu_exchange_gpu.py -x -q > gpurun_out/pytest_dist.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_dist.txt

timeout 900 python -m pytest tests/test_solver.py tests/test_cli.py -q 2>&1 | tail -2 > gpurun_out/log.txt

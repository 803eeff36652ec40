for i in 1 2 3; do timeout 900 python -m pytest tests -m gpu -q -k "reference_unit_tests" 2>&1 | grep -E "FAIL|passed|failed|test_fmm.cpp" | head -5; done > gpurun_out/log.txt 2>&1

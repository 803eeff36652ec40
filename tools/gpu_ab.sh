mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "solve or krylov or adapter or cli" > gpurun_out/pytest_sub.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_sub.txt
./oracle/_ref/adapter_parity > gpurun_out/adapter.txt 2>&1; echo "exit $?" >> gpurun_out/adapter.txt

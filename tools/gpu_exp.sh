for h in 0 1; do echo "HERM=$h"; BLFMM_HERMITIAN=$h python tools/run_steps.py --steps 3 2>&1 | tail -1; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15

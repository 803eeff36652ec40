timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
python tools/time_step.py --tag shared --steps 10
python tools/time_step.py --tag scaled10 --scaled 10 --steps 3

timeout 1500 python -m pytest tests/ -x -q -m gpu -k "not config4" 2>&1 | tail -3

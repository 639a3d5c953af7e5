timeout 2400 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
timeout 300 python tools/quick_time.py c4 c4s c3 c2 c1 c5

# full GPU suite + timing of the defaults
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
timeout 2400 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -4
timeout 300 python tools/quick_time.py c4 c4s c3 c2 c1

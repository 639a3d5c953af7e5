# unconditional-commit rounds in k_zig_tma: parity (lane policy + full C3/C4) and timing
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "lane and not ring" 2>&1 | tail -3
GZ_POLICY=lane timeout 300 python tools/quick_time.py c4 c4s c3
GZ_POLICY=lane timeout 300 python tools/quick_time.py c4 c4s c3

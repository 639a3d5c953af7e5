timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "lane and not tma and not ring" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullconfig.py -x -q -k "config4" 2>&1 | tail -2
GZ_POLICY=lane timeout 300 python tools/quick_time.py c4 c4s c3 | grep -v policy

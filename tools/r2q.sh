python tools/quick_time.py c3 c4 c4s c5 2>&1 | tee gpurun_out/r2q_time.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "random_streams or strided or guard or mutat or config" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullconfig.py -x -q 2>&1 | tail -2

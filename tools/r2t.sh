python tools/quick_time.py c2 2>&1 | tail -1 | tee gpurun_out/r2t_time.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "polar or pairing or config2 or random_streams" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullconfig.py -x -q -k "config2" 2>&1 | tail -2

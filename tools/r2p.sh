python tools/quick_time.py c5 2>&1 | tee gpurun_out/r2p_time.txt
GZ_LIB=build/var/mut14/libgzb200.so python tools/quick_time.py c5 2>&1 | tee -a gpurun_out/r2p_time.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "mutat or config5" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullconfig.py -x -q -k "config5" 2>&1 | tail -2
GZ_LIB=build/var/mut14/libgzb200.so timeout 900 python -m pytest tests/test_gpu_fullconfig.py -x -q -k "config5" 2>&1 | tail -2

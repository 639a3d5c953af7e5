python tools/quick_time.py c5 2>&1 | tee gpurun_out/r2o_time.txt
GZ_POLICY=lane-ring python tools/quick_time.py c5 2>&1 | tee -a gpurun_out/r2o_time.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "mutat or config5" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_fullconfig.py -x -q -k "config5" 2>&1 | tail -3

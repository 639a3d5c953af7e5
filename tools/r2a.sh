set -x
python tools/quick_time.py c3 c4 c4s 2>&1 | tee gpurun_out/r2a_time_auto.txt
GZ_POLICY=lane-ring python tools/quick_time.py c3 c4 c4s 2>&1 | tee gpurun_out/r2a_time_ring.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "random_streams or strided or guard or zero_sizes or custom_layer or config" 2>&1 | tail -15 | tee gpurun_out/r2a_parity.txt
timeout 900 python -m pytest tests/test_gpu_fullconfig.py -x -q -s 2>&1 | tail -25 | tee gpurun_out/r2a_full.txt

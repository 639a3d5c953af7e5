for sh in 0 1 2 3; do echo "shape $sh"; GZ_TMA_SHAPE=$sh python tools/quick_time.py c4 c4s 2>&1 | grep -v policy | tail -2; done | tee gpurun_out/r2h_shapes.txt
for sh in 0 2; do echo "shape $sh"; GZ_TMA_SHAPE=$sh python tools/quick_time.py c3 2>&1 | grep -v policy | tail -1; done | tee -a gpurun_out/r2h_shapes.txt
timeout 600 python -m pytest tests/test_gpu_fullconfig.py -x -q -k "config4 or config3" 2>&1 | tail -3 | tee gpurun_out/r2h_full.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "random_streams or strided or guard or zero_sizes or custom_layer or config" 2>&1 | tail -3 | tee gpurun_out/r2h_parity.txt

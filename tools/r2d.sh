for sh in 0 2 3; do echo "shape $sh"; GZ_TMA_SHAPE=$sh python tools/quick_time.py c3 c4 c4s 2>&1 | grep -v policy; done | tee gpurun_out/r2d_shapes.txt
python tools/prof_one.py c4 0 1 > /dev/null && GZ_TMA_SHAPE=3 ncu --set full --clock-control none --import-source on -k regex:k_zig_tma -c 1 -o gpurun_out/r2d_c4_tma3 python tools/prof_one.py c4 0 1 > gpurun_out/r2d_ncu.log 2>&1
GZ_TMA_SHAPE=3 timeout 600 python -m pytest tests/test_gpu_fullconfig.py -x -q -k "config4 or config3" 2>&1 | tail -3 | tee gpurun_out/r2d_full.txt
GZ_TMA_SHAPE=3 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "random_streams or strided or guard or zero_sizes or custom_layer or config" 2>&1 | tail -3 | tee gpurun_out/r2d_parity.txt

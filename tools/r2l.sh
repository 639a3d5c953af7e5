for sh in 0 2 3; do echo "shape $sh"; GZ_TMA_SHAPE=$sh python tools/quick_time.py c3 c4 c4s 2>&1 | grep -v policy; done | tee gpurun_out/r2l_shapes.txt
GZ_TMA_SHAPE=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullconfig.py -x -q -k "random_streams or strided or guard or config" 2>&1 | tail -2

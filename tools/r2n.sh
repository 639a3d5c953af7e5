for sh in 0 5 6 7 8; do echo "shape $sh"; GZ_TMA_SHAPE=$sh python tools/quick_time.py c4 c4s 2>&1 | grep -v policy; done | tee gpurun_out/r2n_shapes.txt
for sh in 5 8; do GZ_TMA_SHAPE=$sh timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullconfig.py -x -q -k "(random_streams and not modified) or strided or guard or config4" 2>&1 | tail -2; done

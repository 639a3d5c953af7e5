for sh in 0 2 3 4; do echo "shape $sh"; GZ_TMA_SHAPE=$sh python tools/quick_time.py c4 c4s 2>&1 | grep -v policy; done | tee gpurun_out/r2m_shapes.txt

for sh in 0; do echo "shape $sh"; GZ_TMA_SHAPE=$sh python tools/quick_time.py c3 c4 c4s 2>&1 | grep -v policy; done | tee gpurun_out/r2g_shapes.txt
timeout 600 python -m pytest tests/test_gpu_fullconfig.py -x -q -k "config4 or config3" 2>&1 | tail -3 | tee gpurun_out/r2g_full.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "random_streams or strided or guard or zero_sizes or custom_layer or config" 2>&1 | tail -3 | tee gpurun_out/r2g_parity.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; tail -3 gpurun_out/r2g_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2g_bench_ref.json 2> gpurun_out/r2g_bench_ref.err; tail -3 gpurun_out/r2g_bench_ref.err
nproc; free -g | head -2

set -x
python tools/quick_time.py c3 c4 c4s 2>&1 | tee gpurun_out/r2b_time_auto.txt
python tools/prof_one.py c4 0 1 > /dev/null && ncu --set full --clock-control none --import-source on -k regex:k_zig_tma -c 1 -o gpurun_out/r2b_c4_tma python tools/prof_one.py c4 0 1 > gpurun_out/r2b_ncu.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fullconfig.py -x -q -k "config4 or config3" 2>&1 | tail -3 | tee gpurun_out/r2b_full.txt

# k_zig_lst variants: conversion by DADDs (l20) vs I2F (l20i), 24 warps (l24); default build = 16 warps
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "test_random_streams_vs_oracle and lane" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullconfig.py -x -q -k "config3 or config4" 2>&1 | tail -2
echo "== l16"; GZ_POLICY=lane timeout 300 python tools/quick_time.py c4 c4s c3 | grep -v policy
for v in l20 l20i l24; do echo "== $v"; GZ_POLICY=lane GZ_LIB=build/var/$v/libgzb200.so timeout 300 python tools/quick_time.py c4 c4s c3 2>&1 | grep -v policy; done

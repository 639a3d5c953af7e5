# non-volatile table gathers: k_zig_lst (16 warps: DADD / I2F conversion; 20 warps) and k_zig_tma
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "test_random_streams_vs_oracle and lane" 2>&1 | tail -2
echo "== l16"; GZ_POLICY=lane timeout 300 python tools/quick_time.py c4 c4s c3 | grep -v policy
for v in l16i l20 l20i; do echo "== $v"; GZ_POLICY=lane GZ_LIB=build/var/$v/libgzb200.so timeout 300 python tools/quick_time.py c4 c4s c3 2>&1 | grep -v policy; done
echo "== tma"; GZ_POLICY=lane-tma timeout 300 python tools/quick_time.py c4 c4s c3 | grep -v policy

# k_zig_lst: parity (lane policy, full C3/C4 shards) and timing (16 / 12 / 20 warps per SM) vs k_zig_tma
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "lane and not ring and not tma" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_fullconfig.py -x -q -k "config3 or config4" 2>&1 | tail -3
echo "== l16"; GZ_POLICY=lane timeout 300 python tools/quick_time.py c4 c4s c3
for v in l12 l20; do echo "== $v"; GZ_POLICY=lane GZ_LIB=build/var/$v/libgzb200.so timeout 300 python tools/quick_time.py c4 c4s c3 2>&1 | grep -v policy; done
echo "== tma"; GZ_POLICY=lane-tma timeout 300 python tools/quick_time.py c4 c4s c3

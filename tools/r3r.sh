# k_zig_lst attempts per round: 8 (default, 20 warps), 12 and 16 at 20 and 16 warps
timeout 600 python -m pytest tests/test_gpu_fullconfig.py -x -q -k "config4" 2>&1 | tail -1
for v in k12 k16 k16w16 k12w16; do echo "== $v"; GZ_LIB=build/var/$v/libgzb200.so timeout 600 python -m pytest tests/test_gpu_fullconfig.py -x -q -k "config4 and 0" 2>&1 | tail -1; GZ_POLICY=lane GZ_LIB=build/var/$v/libgzb200.so timeout 300 python tools/quick_time.py c4 c4s c3 2>&1 | grep -v policy; done
echo "== k8"; GZ_POLICY=lane timeout 300 python tools/quick_time.py c4 c4s c3 | grep -v policy

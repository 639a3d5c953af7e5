# where k_zig_lst's time goes: without the frozen pass (e1), without row stores (e2), neither (e3)
for v in l20i e1 e2 e3; do echo "== $v"; GZ_POLICY=lane GZ_LIB=build/var/$v/libgzb200.so timeout 300 python tools/quick_time.py c4 c3 2>&1 | grep -v policy; done

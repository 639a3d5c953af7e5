for v in x3 x3w16 x7 x7w16; do echo "== $v"; GZ_POLICY=lane GZ_LIB=build/var/$v/libgzb200.so timeout 300 python tools/quick_time.py c4 2>&1 | grep -v policy; done

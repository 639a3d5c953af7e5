# window-kernel warps-per-SM variants vs the TMA kernel (c4, c4 + witnesses, c3)
for v in w32 w24 w16; do echo "== $v"; GZ_POLICY=win GZ_LIB=build/var/$v/libgzb200.so timeout 300 python tools/quick_time.py c4 c4s c3 2>&1 | grep -v policy; done
echo "== tma"; GZ_POLICY=lane timeout 300 python tools/quick_time.py c4 c4s c3 2>&1 | grep -v policy

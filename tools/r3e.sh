# LCG draw chains in the k_zig_tma UNCOND rounds: parity of the default build, timing of ch1/ch2/ch4
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "lane and not ring" 2>&1 | tail -3
for v in ch1 ch2 ch4; do echo "== $v"; for r in 1 2; do GZ_POLICY=lane GZ_LIB=build/var/$v/libgzb200.so timeout 300 python tools/quick_time.py c4 c4s c3 2>&1 | grep -v policy; done; done

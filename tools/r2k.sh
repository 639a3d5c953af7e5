for v in lseg4; do echo "== $v"; for r in 1 2; do GZ_LIB=build/var/$v/libgzb200.so python tools/quick_time.py c1 2>&1 | grep -v policy; done; done
echo "== default"; for r in 1 2; do python tools/quick_time.py c1 2>&1 | grep -v policy; done
for P in 4 2; do echo "== P=$P"; GZ_LSEG_P=$P python tools/quick_time.py c1 2>&1 | grep -v policy; GZ_LSEG_P=$P GZ_LIB=build/var/lseg4/libgzb200.so python tools/quick_time.py c1 2>&1 | grep -v policy; done

python tools/cmp_policies.py lane lane-tma
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "tma" 2>&1 | tail -1
for r in 1 2; do GZ_POLICY=lane-tma timeout 300 python tools/quick_time.py c4 c4s | grep -v policy; done

set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "win" 2>&1 | tail -15
for pol in win lane; do GZ_POLICY=$pol timeout 300 python tools/quick_time.py c4 c4s c3; done

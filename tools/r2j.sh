# in-kernel self-checks (debug build) over every kernel family: the compute-sanitizer stand-in
export GZ_LIB=$PWD/paper_2405_19493_b200/libgzb200_dbg.so
mkdir -p gpurun_out/selfcheck
for c in tma ring warp lseg single polarq polarlane mutate; do
  timeout 600 python tools/sanitize_cases.py $c > gpurun_out/selfcheck/$c.log 2>&1; echo "$c rc=$? $(tail -1 gpurun_out/selfcheck/$c.log)"
done | tee gpurun_out/selfcheck/summary.txt
timeout 600 python tools/quick_time.py c3 c4 c4s c2 c5 2>&1 | tee gpurun_out/selfcheck/full_size.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullconfig.py -x -q 2>&1 | tail -3 | tee gpurun_out/selfcheck/pytest_dbg.log
timeout 400 python tools/fuzz_gpu.py 240 2468 > gpurun_out/selfcheck/fuzz_dbg.log 2>&1; tail -3 gpurun_out/selfcheck/fuzz_dbg.log

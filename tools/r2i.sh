# compute-sanitizer over every kernel family, the new tests, the full GPU suite, an ncu capture of the C4 headline kernel
mkdir -p gpurun_out/san
for c in tma ring warp lseg single polarq polarlane mutate; do
  for tool in memcheck racecheck synccheck; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py $c > gpurun_out/san/${c}_${tool}.log 2>&1
    echo "$c $tool rc=$? $(tail -1 gpurun_out/san/${c}_${tool}.log)"
  done
done | tee gpurun_out/san/summary.txt
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_fullconfig.py -x -q -s 2>&1 | tail -20 | tee gpurun_out/r2i_multi_full.txt
timeout 1800 python -m pytest tests -x -q -m gpu 2>&1 | tail -5 | tee gpurun_out/r2i_gpu_suite.txt
python bench.py --steps 2 --warmup 3 --no-extra --no-cpu --no-e2e > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_zig_tma -s 3 -c 1 -o gpurun_out/r2i_c4_tma_stats python bench.py --steps 1 --warmup 3 --no-extra --no-cpu --no-e2e > gpurun_out/r2i_ncu.log 2>&1

#!/bin/bash
# Round-2 profiling pass: PART=1: bench line (both arms), launch list of the same bench
# command, `ncu --set full` of the headline kernel; PART=2: one `ncu --set full` capture per
# other config kernel.  Every profiled command first runs to completion without ncu.
# Usage: bash tools/prof_r2.sh TAG PART   (two calls: gpurun brings back <= 64 MiB each)
set -x
TAG=${1:-r2b}
PART=${2:-1}
mkdir -p gpurun_out/$TAG
O=gpurun_out/$TAG
if [ "$PART" = 1 ]; then
python bench.py --steps 20 --warmup 3 > $O/bench.json 2>$O/bench.err || exit 1
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2>$O/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_zig_tma -s 3 -c 1 -o $O/c4_k_zig_tma python bench.py --steps 1 --warmup 3 --no-extra --no-cpu --no-e2e > /dev/null 2>&1
else
python tools/prof_one.py c3 0 1 && ncu --set full --clock-control none --import-source on -k regex:k_zig_tma -c 1 -o $O/c3_k_zig_tma python tools/prof_one.py c3 0 1 > /dev/null 2>&1
python tools/prof_one.py c2 0 1 && ncu --set full --clock-control none --import-source on -k regex:k_polar_q -c 1 -o $O/c2_k_polar_q python tools/prof_one.py c2 0 1 > /dev/null 2>&1
python tools/prof_one.py c5 0 1 && ncu --set full --clock-control none --import-source on -k regex:k_zig_lane -c 1 -o $O/c5_k_zig_lane_mutate python tools/prof_one.py c5 0 1 > /dev/null 2>&1
python tools/prof_one.py c1 0 1 && ncu --set full --clock-control none --import-source on -k regex:k_zig -c 1 -o $O/c1_k_zig_lseg python tools/prof_one.py c1 0 1 > /dev/null 2>&1
fi
ls -la $O

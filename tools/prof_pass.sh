#!/bin/bash
# One profiling pass on the GPU box (every profiled command first runs to completion without ncu):
#   PART=1: the bench line of both arms, the launch list of the bench command, `ncu --set full`
#           of the headline kernel (config 4) and its traffic record (profiles/traffic.json entry);
#   PART=2: one `ncu --set full --clock-control none` capture per other config kernel.
# Summaries are made on the box and the reports dropped (gpurun brings back <= 64 MiB).
# Usage: bash tools/prof_pass.sh TAG PART
set -x
TAG=${1:-r4a}
PART=${2:-1}
O=gpurun_out/$TAG
mkdir -p $O
summ() {  # summ NAME: summaries of $O/NAME.ncu-rep, then drop the report
  python tools/ncu_summary.py $O/$1.ncu-rep > $O/${1}_summary.txt
  ncu -i $O/$1.ncu-rep --page source --print-source sass --csv > $O/$1_src.csv 2>/dev/null
  python tools/sass_hot.py $O/$1_src.csv 30 > $O/${1}_sass_hot.txt
  python tools/sass_blocks.py $O/$1_src.csv 0.003 > $O/${1}_blocks.txt
  python tools/stall_lines.py $O/$1_src.csv 30 > $O/${1}_stalls.txt
  rm -f $O/$1_src.csv $O/$1.ncu-rep
}
cap() {  # cap NAME KERNEL_REGEX CFG (prof_one.py config, trailing s: with the fused witnesses)
  python tools/prof_one.py $3 0 1 > /dev/null && ncu --set full --clock-control none --import-source on -k regex:$2 -c 1 -o $O/$1 python tools/prof_one.py $3 0 1 > /dev/null 2>&1
  summ $1
}
if [ "$PART" = 1 ]; then
  python bench.py --steps 20 --warmup 3 > $O/bench.json 2>$O/bench.err || exit 1
  python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2>$O/bench_ref.err
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_zig_lst -s 3 -c 1 -o $O/c4_k_zig_lst python bench.py --steps 1 --warmup 3 --no-extra --no-cpu --no-e2e > /dev/null 2>&1
  python tools/traffic_record.py $O/c4_k_zig_lst.ncu-rep c4 1073741824 "profiles/$TAG/c4_k_zig_lst_summary.txt (ncu --set full --clock-control none, bench.py --no-extra, 4th launch)" > $O/traffic_c4.json
  cp profiles/traffic.json $O/traffic.json
  summ c4_k_zig_lst
else
  cap c3_k_zig_lst k_zig_lst c3
  cap c2_k_polar_lst k_polar_lst c2
  cap c5_k_zig_lst_mutate k_zig_lst c5
  cap c1_k_zig_lseg k_zig_lseg c1
fi
ls -la $O

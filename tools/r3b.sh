# ncu capture of the window kernel (c4 with witnesses) and the TMA kernel, summaries on the box
set -x
O=gpurun_out/r3b; mkdir -p $O
cap() {  # cap NAME KERNEL_REGEX CFG POLICY
  GZ_POLICY=$4 python tools/prof_one.py $3 0 1 > /dev/null && GZ_POLICY=$4 ncu --set full --clock-control none --import-source on -k regex:$2 -c 1 -o $O/$1 python tools/prof_one.py $3 0 1 > /dev/null 2>&1
  python tools/ncu_summary.py $O/$1.ncu-rep > $O/${1}_summary.txt
  ncu -i $O/$1.ncu-rep --page source --print-source sass --csv > $O/$1_src.csv 2>/dev/null
  python tools/sass_hot.py $O/$1_src.csv 40 > $O/${1}_sass_hot.txt
  python tools/sass_blocks.py $O/$1_src.csv 0.002 > $O/${1}_blocks.txt
  rm -f $O/$1.ncu-rep
}
cap c4_win k_zig_win c4 win
cap c4_tma k_zig_tma c4 lane
ls -la $O

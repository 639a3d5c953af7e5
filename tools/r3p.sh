set -x
O=gpurun_out/r3p; mkdir -p $O
cap() {  # cap NAME KERNEL_REGEX CFG POLICY [LIB]
  GZ_LIB=$5 GZ_POLICY=$4 python tools/prof_one.py $3 0 1 > /dev/null && GZ_LIB=$5 GZ_POLICY=$4 ncu --set full --clock-control none --import-source on -k regex:$2 -c 1 -o $O/$1 python tools/prof_one.py $3 0 1 > /dev/null 2>&1
  python tools/ncu_summary.py $O/$1.ncu-rep > $O/${1}_summary.txt
  ncu -i $O/$1.ncu-rep --page source --print-source sass --csv > $O/$1_src.csv 2>/dev/null
  python tools/sass_blocks.py $O/$1_src.csv 0.002 > $O/${1}_blocks.txt
  python tools/stall_lines.py $O/$1_src.csv 40 > $O/${1}_stalls.txt
  rm -f $O/$1.ncu-rep
}
cap c4_x3 k_zig_lst c4 lane build/var/x3/libgzb200.so
cap c4_lst k_zig_lst c4 lane

set -x
TAG=${1:-r1f}
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench.json 2>gpurun_out/${TAG}_bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_polar_q -s 3 -c 1 -o gpurun_out/${TAG}_c2_k_polar_q python bench.py --steps 1 --warmup 3 --no-extra --no-cpu > /dev/null 2>&1
python tools/prof_one.py c3 0 1 && ncu --set full --clock-control none --import-source on -k regex:k_zig_lane -c 1 -o gpurun_out/${TAG}_c3_k_zig_lane python tools/prof_one.py c3 0 1 > /dev/null 2>&1
python tools/prof_one.py c4 0 1 && ncu --set full --clock-control none --import-source on -k regex:k_zig_lane -c 1 -o gpurun_out/${TAG}_c4_k_zig_lane python tools/prof_one.py c4 0 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_zig_lane -c 1 -o gpurun_out/${TAG}_c5_k_zig_lane_mutate python tools/prof_one.py c5 0 1 > /dev/null 2>&1
python tools/prof_one.py c1 0 1 && ncu --set full --clock-control none --import-source on -k regex:k_zig -c 1 -o gpurun_out/${TAG}_c1_k_zig python tools/prof_one.py c1 0 1 > /dev/null 2>&1
python tools/one_single.py ziggurat splitmix 24 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_single_zig_launches.csv python tools/one_single.py ziggurat splitmix 24 > /dev/null 2>&1
python tools/one_single.py polar lcg48 24 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_single_polar_launches.csv python tools/one_single.py polar lcg48 24 > /dev/null 2>&1
ls -la gpurun_out/

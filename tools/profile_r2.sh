#!/bin/bash
# Sweep evidence behind bench.py's roofline, one GPU (round 2):  $1 = tag.
# Writes gpurun_out/prof_$1/: launch list of 2 V-cycles, DRAM bytes + time of
# every sweep launch of one V-cycle (cold L2 per launch), and ncu --set full of
# the first 14 sweep launches (level-1 first forward half-sweep + the
# following backward phases).  bench.py --profile-only must have exited 0
# (run it before this script in the same gpurun call).
set -u
T=${1:-cur}
O=gpurun_out/prof_$T
mkdir -p $O
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches.csv python bench.py --profile-only --steps 2 > $O/ncu_l.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 14 -f -o $O/sweep_full \
    python bench.py --profile-only --steps 1 > $O/ncu_f.log 2>&1; echo full=$?
ncu -i $O/sweep_full.ncu-rep --page raw --csv > $O/sweep_full_raw.csv 2>/dev/null; echo raw=$?
ncu -i $O/sweep_full.ncu-rep --page source --csv > $O/sweep_full_source.csv 2>/dev/null; echo src=$?

#!/bin/bash
# The sweep evidence behind bench.py's roofline (profiles/README.md), one GPU:
#   $1 = tag.  Writes gpurun_out/{launches,sweep_dram,sweep_full_raw}_$1.csv
# 1. launch list of bench.py --profile-only (2 V-cycles): per-kernel shares
# 2. DRAM bytes of every sweep launch of one V-cycle (cold L2 per launch)
# 3. ncu --set full of the first 6 sweep launches (level-1 forward half-sweep)
set -u
T=${1:-cur}
O=gpurun_out
mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$T.csv \
    python bench.py --profile-only > $O/ncu_l_$T.log 2>&1; echo launches=$?
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_sweep -c 134 --csv --log-file $O/sweep_dram_$T.csv \
    python bench.py --profile-only > $O/ncu_d_$T.log 2>&1; echo dram=$?
ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 6 -f -o $O/sweep_full_$T \
    python bench.py --profile-only > $O/ncu_f_$T.log 2>&1; echo full=$?
ncu -i $O/sweep_full_$T.ncu-rep --page raw --csv > $O/sweep_full_raw_$T.csv 2>/dev/null; echo raw=$?

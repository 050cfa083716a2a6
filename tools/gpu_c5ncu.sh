#!/bin/bash
# C5 (round tags): launch list of one solve + ncu --set full of one mid-solve phase-3 launch
mkdir -p gpurun_out/c5n
O=gpurun_out/c5n
# (launch list captured once) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_c5.csv python tools/solve_once.py --config C5 > $O/ncu_list.log 2>&1
# python tools/launch_summary.py $O/launches_c5.csv > $O/launches_c5_summary.txt 2>&1
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base mangled"
timeout 900 $NCU -k regex:'minplus_tile_kernelIfLi128ELi128ELi1ELb0E' --launch-skip 128 --launch-count 1 -f -o $O/p3_c5 python tools/solve_once.py --config C5 > $O/ncu_p3.log 2>&1
python tools/ncu_summary.py $O/p3_c5.ncu-rep > $O/p3_c5_summary.txt 2>&1

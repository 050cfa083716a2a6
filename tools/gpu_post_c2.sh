#!/bin/bash
# Post-pass evidence at C2 / C5: launch list of one solve, ncu --set full of the resolve and finalize.
O=gpurun_out/post
R=/tmp/post_reps
mkdir -p $O $R
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python tools/solve_once.py --config C2 --reps 2 > $O/list_c2.log 2>&1
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base mangled"
timeout 600 $NCU -k regex:'resolve_lastk' --launch-skip 1 --launch-count 1 -f -o $R/res_c2 python tools/solve_once.py --config C2 --reps 2 > $O/ncu_res.log 2>&1
python tools/ncu_summary.py $R/res_c2.ncu-rep > $O/res_c2_summary.txt 2>&1
ncu -i $R/res_c2.ncu-rep --page source --csv > $O/res_c2_source.csv 2>/dev/null
timeout 600 $NCU -k regex:'finalize_paths' --launch-skip 1 --launch-count 1 -f -o $R/fin_c2 python tools/solve_once.py --config C2 --reps 2 > $O/ncu_fin.log 2>&1
python tools/ncu_summary.py $R/fin_c2.ncu-rep > $O/fin_c2_summary.txt 2>&1
timeout 600 $NCU -k regex:'transpose' --launch-skip 1 --launch-count 1 -f -o $R/tr_c2 python tools/solve_once.py --config C2 --reps 2 > $O/ncu_tr.log 2>&1
python tools/ncu_summary.py $R/tr_c2.ncu-rep > $O/tr_c2_summary.txt 2>&1

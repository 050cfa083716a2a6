#!/bin/bash
# Round-2 evidence: GPU tests, smoke, bench lines (C4 headline with CPU baseline + ladder, C5, C3,
# C2, N=65536), C4 launch list, ncu --set full of the dominant kernels of the current build:
# the C4 bulk launch (KEY, 256-deep), a C5 round-tag launch, phase 1 (FP32 keys) and the dual
# phase-2 launch at C4, and the persistent kernel at C2 (one whole solve).
O=gpurun_out/ev2
R=/tmp/ev2_reps   # ncu reports stay on the box (gpurun copies back at most 64 MiB): summaries only
mkdir -p $O $R
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --e2e-steps 3 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --config C5 --no-cpu > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --config C3 --no-cpu --e2e-steps 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config C2 --no-cpu --e2e-steps 3 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 1200 python bench.py --n 65536 --steps 1 --warmup 1 --no-e2e --no-cpu --no-isolated > $O/bench_n65536.json 2> $O/bench_n65536.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/reference_arm.json 2> $O/reference_arm.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $R/launches_c4.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-isolated > $O/ncu_list.log 2>&1
python tools/launch_summary.py $R/launches_c4.csv > $O/launches_c4_summary.txt 2>&1
gzip -c $R/launches_c4.csv > $O/launches_c4.csv.gz
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base mangled"
timeout 600 $NCU -k regex:'minplus_tile_kernelIfLi128ELi128ELi2ELb0E' --launch-skip 40 --launch-count 1 -f -o $R/p3_c4 python tools/solve_once.py --config C4 > $O/ncu_p3.log 2>&1
python tools/ncu_summary.py $R/p3_c4.ncu-rep > $O/p3_c4_summary.txt 2>&1
ncu -i $R/p3_c4.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv, sys, json
rows = list(csv.reader(sys.stdin))
h, u, v = rows[0], rows[1], rows[2]
keep = {k: v[i] for i, k in enumerate(h) if k.startswith(('dram__bytes', 'gpu__time_duration', 'smsp__inst_executed.sum', 'sm__cycles_elapsed'))}
json.dump(keep, open('$O/p3_c4_raw_keys.json', 'w'), indent=1)"
timeout 900 $NCU -k regex:'minplus_tile_kernelIfLi128ELi128ELi1ELb0E' --launch-skip 128 --launch-count 1 -f -o $R/p3_c5 python tools/solve_once.py --config C5 > $O/ncu_p3c5.log 2>&1
python tools/ncu_summary.py $R/p3_c5.ncu-rep > $O/p3_c5_summary.txt 2>&1
timeout 600 $NCU -k regex:'phase1_key_f32_kernel' --launch-skip 40 --launch-count 1 -f -o $R/p1_c4 python tools/solve_once.py --config C4 > $O/ncu_p1.log 2>&1
python tools/ncu_summary.py $R/p1_c4.ncu-rep > $O/p1_c4_summary.txt 2>&1
FW_PAIRS=0 timeout 600 $NCU -k regex:'minplus_tile_kernelIfLi128ELi128ELi2ELb1E' --launch-skip 40 --launch-count 1 -f -o $R/p2_c4 python tools/solve_once.py --config C4 > $O/ncu_p2.log 2>&1
python tools/ncu_summary.py $R/p2_c4.ncu-rep > $O/p2_c4_summary.txt 2>&1
timeout 600 $NCU -k regex:'fw_persistent_kernel' --launch-count 1 -f -o $R/persist_c2 python tools/solve_once.py --config C2 > $O/ncu_persist.log 2>&1
python tools/ncu_summary.py $R/persist_c2.ncu-rep > $O/persist_c2_summary.txt 2>&1

#!/bin/bash
# Phase 1 with two steps per barrier: full GPU tests, C2/C3/C4 bench lines, isolated phase-1 times.
mkdir -p gpurun_out/p1
O=gpurun_out/p1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python bench.py --config C2 --no-cpu --e2e-steps 3 --steps 20 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config C3 --no-cpu --e2e-steps 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --no-cpu --e2e-steps 3 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:phase1 -c 200 --csv --log-file $O/p1_c2.csv python tools/solve_once.py --config C2 > $O/ncu.log 2>&1
python tools/launch_summary.py $O/p1_c2.csv > $O/p1_c2_summary.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:phase1 -c 200 --csv --log-file $O/p1_c4.csv python tools/solve_once.py --config C4 > $O/ncu4.log 2>&1
python tools/launch_summary.py $O/p1_c4.csv > $O/p1_c4_summary.txt 2>&1

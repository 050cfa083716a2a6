#!/bin/bash
O=gpurun_out/stage2
mkdir -p $O
timeout 600 python tools/ab_options.py --config C2 --sets "persist_gap=-1;persist_gap=400;persist_gap=500;persist_gap=600;persist_gap=-1;persist_gap=500;persist_quarters=0,persist_gap=500" --reps 15 > $O/ab_c2.jsonl 2>&1
timeout 600 python tools/ab_options.py --config C2 --n 3072 --sets "persist_gap=-1;persist_gap=300;persist_gap=500;persist_quarters=2" --reps 15 > $O/ab_n3072.jsonl 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_all.log 2>&1; echo "pytest rc=$?" >> $O/pytest_all.log
timeout 600 python bench.py --config C2 --no-cpu --e2e-steps 3 --steps 20 > $O/bench_c2.json 2> $O/bench_c2.err

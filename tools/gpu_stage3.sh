#!/bin/bash
O=gpurun_out/stage3
mkdir -p $O
timeout 600 python tools/ab_options.py --config C2 --sets "persist_gap=-1;persist_gap=550;persist_gap=600;persist_gap=650;persist_gap=600;persist_gap=-1" --reps 15 > $O/ab_c2.jsonl 2>&1
timeout 600 python tools/ab_options.py --config C2 --n 2048 --sets "persist_quarters=1;persist_quarters=2;persist_quarters=1;persist_quarters=2" --reps 15 > $O/ab_n2048.jsonl 2>&1
timeout 600 python tools/ab_options.py --config C2 --n 1024 --sets "persist_quarters=1;persist_quarters=2;persistent=0" --reps 15 > $O/ab_n1024.jsonl 2>&1
timeout 600 python tools/ab_options.py --config C2 --n 3072 --sets "persist_quarters=1;persist_quarters=2" --reps 15 > $O/ab_n3072.jsonl 2>&1

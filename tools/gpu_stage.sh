#!/bin/bash
O=gpurun_out/stage
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -q -x -k "persist or C2 or tag or real" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python tools/ab_options.py --config C2 --sets "persist_stage_old=0;persist_stage_old=1;persist_stage_old=0;persist_stage_old=1;persist_stage_old=1,persist_quarters=0;persist_stage_old=1,persist_gap=500" --reps 15 > $O/ab_c2.jsonl 2>&1
timeout 600 python tools/ab_options.py --config C2 --n 2048 --sets "persist_stage_old=0;persist_stage_old=1" --reps 15 > $O/ab_n2048.jsonl 2>&1
timeout 600 python tools/ab_options.py --config C3 --sets "persistent=1,persist_stage_old=0;persistent=1,persist_stage_old=1" --reps 5 > $O/ab_c3.jsonl 2>&1
FW_PERSIST_TRACE=/tmp/tr.bin timeout 120 python tools/solve_once.py --config C2 --reps 3 > $O/solve.log 2>&1
python tools/persist_trace.py /tmp/tr.bin --n 4096 > $O/trace.json 2>&1

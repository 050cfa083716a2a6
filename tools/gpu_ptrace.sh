#!/bin/bash
# Persistent-kernel item traces at C2 (default options, and quarters off / gap variants).
O=gpurun_out/ptrace
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "C2 or tag or real" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python tools/ab_options.py --config C2 --sets "persistent=1;persistent=1" --reps 9 > $O/ab_c2.jsonl 2>&1
FW_PERSIST_TRACE=/tmp/tr_c2.bin timeout 120 python tools/solve_once.py --config C2 --reps 3 > $O/solve.log 2>&1
python tools/persist_trace.py /tmp/tr_c2.bin --n 4096 > $O/trace_c2.json 2>&1
FW_PERSIST_TRACE=/tmp/tr_c3.bin FW_PERSISTENT=1 timeout 120 python tools/solve_once.py --config C3 --reps 2 > $O/solve3.log 2>&1
python tools/persist_trace.py /tmp/tr_c3.bin --n 8192 > $O/trace_c3.json 2>&1
cp /tmp/tr_c2.bin $O/

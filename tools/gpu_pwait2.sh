#!/bin/bash
O=gpurun_out/pwait2
mkdir -p $O
FW_PERSIST_TRACE=/tmp/tr.bin timeout 120 python tools/solve_once.py --config C2 --reps 3 > $O/solve.log 2>&1
python tools/persist_trace.py /tmp/tr.bin --n 4096 > $O/trace.json 2>&1

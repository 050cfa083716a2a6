#!/bin/bash
mkdir -p gpurun_out/pp
O=gpurun_out/pp
for r in 8 16 32; do
  FW_PIPE_PAIR_ROWS=$r timeout 600 python tools/pipe_probe.py --config C4 --chunks=-1 --reps 2 > $O/c4_$r.log 2>&1
  FW_PIPE_PAIR_ROWS=$r timeout 600 python tools/pipe_probe.py --config C3 --chunks=-1 --reps 2 > $O/c3_$r.log 2>&1
done

#!/bin/bash
mkdir -p gpurun_out/pf
O=gpurun_out/pf
for f in 4 8 16 32; do
  FW_PIPE_FIRST=$f timeout 600 python tools/pipe_probe.py --config C4 --chunks=-1 --reps 2 > $O/c4_$f.log 2>&1
done

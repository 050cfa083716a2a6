#!/bin/bash
# host pipeline geometry after the pair overlap: first chunk x smallest paired chunk (C4, C3)
mkdir -p gpurun_out/ps
O=gpurun_out/ps
for cfg in C4 C3; do
  for f in 4 8; do
    for pr in 16 32; do
      FW_PIPE_FIRST=$f FW_PIPE_PAIR_ROWS=$pr timeout 600 python tools/pipe_probe.py --config $cfg --chunks=-1 --reps 3 > $O/${cfg}_f${f}_p${pr}.log 2>&1
    done
  done
done

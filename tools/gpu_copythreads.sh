#!/bin/bash
mkdir -p gpurun_out/ct
for t in 3 7 11 15; do
  FW_COPY_THREADS=$t timeout 600 python tools/pipe_probe.py --config C4 --chunks=-1 --reps 2 --pageable > gpurun_out/ct/c4_$t.log 2>&1
done
nproc > gpurun_out/ct/nproc.txt

#!/bin/bash
# A/B of the blocked phase 1 (FW_P1_BLOCKED=0/1): every GPU test with the blocked phase 1 (the
# default), then isolated / in-solve timings at C2 (round tags), C4 (FP32 keys) and C5.
O=gpurun_out/r2n
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for B in 0 1; do
  for c in C2 C4; do
    FW_P1_BLOCKED=$B timeout 600 python tools/ab_options.py --config $c --sets "lookahead=0,pairs=0,persistent=0;persistent=-1" --reps 3 | sed "s/^/{\"p1_blocked\": $B, \"r\": /; s/$/}/" >> $O/ab.jsonl 2>>$O/ab.err
  done
done

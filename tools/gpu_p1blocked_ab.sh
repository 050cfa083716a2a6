#!/bin/bash
# A/B of the blocked phase 1 (FW_P1_BLOCKED) and the rewritten TAG resolve: parity tests of the
# round-tag paths, then isolated / in-solve timings at C2 and C5.
O=gpurun_out/r2m
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_pipeline.py -q -p no:cacheprovider -x -k "real or C2 or tag or TAG or persistent or lastk or loopback or er_f32 or pipeline" > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for B in 0 1; do
  for c in C2 C5; do
    FW_P1_BLOCKED=$B timeout 600 python tools/ab_options.py --config $c --sets "lookahead=0,pairs=0,persistent=0;persistent=0;persistent=-1" --reps 3 | sed "s/^/{\"p1_blocked\": $B, \"r\": /; s/$/}/" >> $O/ab.jsonl 2>>$O/ab.err
  done
done

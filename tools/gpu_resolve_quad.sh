#!/bin/bash
# Quad-lane resolve + stream-mirroring loopback: parity tests, A/B at C2 / C5, ncu of the new resolve.
O=gpurun_out/rq
R=/tmp/rq_reps
mkdir -p $O $R
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python tools/ab_options.py --config C2 --sets "resolve_quad=0;resolve_quad=1;resolve_quad=0;resolve_quad=1" --reps 9 > $O/ab_c2.jsonl 2>&1
timeout 600 python tools/ab_options.py --config C5 --sets "resolve_quad=0;resolve_quad=1" --reps 2 > $O/ab_c5.jsonl 2>&1
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base mangled"
timeout 600 $NCU -k regex:'resolve_lastk_quad' --launch-skip 1 --launch-count 1 -f -o $R/resq_c2 python tools/solve_once.py --config C2 --reps 2 > $O/ncu_resq.log 2>&1
python tools/ncu_summary.py $R/resq_c2.ncu-rep > $O/resq_c2_summary.txt 2>&1

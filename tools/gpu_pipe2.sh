#!/bin/bash
mkdir -p gpurun_out/pipe
O=gpurun_out/pipe
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_all.log 2>&1; echo "pytest rc=$?" >> $O/pytest_all.log
timeout 900 python tools/pipe_probe.py --config C4 --chunks 0,-1 --reps 2 --pageable > $O/probe_c4_pageable.log 2>&1
timeout 900 python tools/pipe_probe.py --config C2 --chunks 0 --reps 3 --pageable > $O/probe_c2_pageable.log 2>&1

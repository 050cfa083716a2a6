#!/bin/bash
O=gpurun_out/lone2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -q -x -k "persist or C2 or tag or real" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python tools/ab_options.py --config C2 --sets "persist_p1_lone=-1;persist_p1_lone=0;persist_p1_lone=-1" --reps 15 > $O/ab_c2.jsonl 2>&1
FW_PERSIST_TRACE=/tmp/tr.bin timeout 120 python tools/solve_once.py --config C2 --reps 3 > $O/solve.log 2>&1
python tools/persist_trace.py /tmp/tr.bin --n 4096 > $O/trace.json 2>&1
timeout 600 python bench.py --config C2 --no-cpu --e2e-steps 3 --steps 20 > $O/bench_c2.json 2> $O/bench_c2.err

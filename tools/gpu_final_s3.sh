#!/bin/bash
O=gpurun_out/fs3
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_all.log 2>&1; echo "pytest rc=$?" >> $O/pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py --config C2 --no-cpu --e2e-steps 3 --steps 20 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 300 python tools/ab_options.py --config C2 --sets "persistent=1;persistent=0" --reps 15 > $O/ab_c2.jsonl 2>&1
FW_PERSIST_TRACE=/tmp/tr.bin timeout 120 python tools/solve_once.py --config C2 --reps 3 > $O/solve.log 2>&1
python tools/persist_trace.py /tmp/tr.bin --n 4096 > $O/trace_c2.json 2>&1

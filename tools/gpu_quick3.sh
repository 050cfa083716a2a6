#!/bin/bash
# Full GPU tests + C4 bench line + launch list summary.
mkdir -p gpurun_out/q
O=gpurun_out/q
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python bench.py --no-cpu --e2e-steps 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench rc=$?" >> $O/bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_c4.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $O/ncu_list.log 2>&1
python tools/launch_summary.py $O/launches_c4.csv > $O/launches_c4_summary.txt 2>&1

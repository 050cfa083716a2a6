#!/bin/bash
mkdir -p gpurun_out/fin
O=gpurun_out/fin
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python bench.py --e2e-steps 3 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --config C5 --no-cpu > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --config C3 --no-cpu --e2e-steps 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config C2 --no-cpu --e2e-steps 3 --steps 20 > $O/bench_c2.json 2> $O/bench_c2.err

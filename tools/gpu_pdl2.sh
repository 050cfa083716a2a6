#!/bin/bash
# programmatic serialization in the single-round look-ahead too: full GPU suite, C2 / C5 / C4 on / off
mkdir -p gpurun_out/pdl2
O=gpurun_out/pdl2
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for o in 1 0 1 0; do
  FW_PDL=$o timeout 300 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu --e2e-steps 3 >> $O/c2_$o.jsonl 2>> $O/err.log
done
for o in 1 0; do
  FW_PDL=$o timeout 600 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu --no-e2e >> $O/c5_$o.jsonl 2>> $O/err.log
  FW_PDL=$o FW_PAIRS=0 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e >> $O/c4single_$o.jsonl 2>> $O/err.log
done

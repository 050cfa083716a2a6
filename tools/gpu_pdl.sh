#!/bin/bash
# bulk launches with programmatic serialization (FW_PDL=1) vs stream order (0)
mkdir -p gpurun_out/pdl
O=gpurun_out/pdl
timeout 900 python -m pytest tests -m gpu -x -q -k "pair or fuzz or pipeline or C4 or C3" > $O/pytest.log 2>&1
for o in 1 0 1 0; do
  FW_PDL=$o timeout 300 python bench.py --steps 5 --warmup 3 >> $O/c4_$o.jsonl 2>> $O/err.log
done
for o in 1 0; do
  FW_PDL=$o timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu >> $O/c3_$o.jsonl 2>> $O/err.log
done

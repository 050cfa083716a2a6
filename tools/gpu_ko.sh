#!/bin/bash
# quick A/B of a rebuilt library: C4 / C5 / C2 / C3 device-resident lines + parity smoke
O=gpurun_out/ko${1:-}
mkdir -p $O
timeout 300 python bench.py --config C4 --no-cpu --no-e2e --no-isolated --steps 5 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 300 python bench.py --config C5 --no-cpu --no-e2e --no-isolated --steps 3 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 300 python bench.py --config C2 --no-cpu --no-e2e --no-isolated --steps 20 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 300 python bench.py --config C3 --no-cpu --no-e2e --no-isolated --steps 5 > $O/bench_c3.json 2> $O/bench_c3.err
for c in c4 c5 c2 c3; do python - <<PY
import json
try:
    d=json.load(open("$O/bench_$c.json")); print("$c", round(d["value"]), "GFLOPS", round(d["ms_per_step"],2), "ms", d["roofline"]["phase_ms_per_step"])
except Exception as e: print("$c", "failed", e)
PY
done

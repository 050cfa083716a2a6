"""A/B of schedule options (fw_set_option) on a device-resident solve of a BASELINE config:
python tools/ab_options.py --config C2 --sets "persistent=0;persistent=1,persist_gap=300" --reps 5
Prints one JSON line per option set: median solve ms and 2n^3/t TFLOPS."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import apsp_inputs as gen  # noqa: E402
import paper_1811_01201_b200 as fw  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--sets", default="persistent=0;persistent=1")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--nopath", action="store_true")
a = ap.parse_args()
c = dict(gen.CONFIGS[a.config])
n = a.n or c["n"]
dW = gen.generate_torch(c["kind"], n, c["seed"], device="cuda", p=c.get("p", 1.0), lo=c.get("lo", 1),
                        hi=c.get("hi", 100))
dD = torch.empty_like(dW)
dP = None if a.nopath else torch.empty(dW.shape, dtype=torch.int32, device="cuda")
f = fw.fw_solve_device_i32 if dW.dtype == torch.int32 else fw.fw_solve_device_f32
for spec in a.sets.split(";"):
    fw.fw_init(0, fw.FW_TIMING)
    opts = {}
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        opts[k] = int(v)
        fw.fw_set_option(k, int(v))
    ms, st = [], None
    for r in range(a.reps + 1):
        dD.copy_(dW)
        f(dD, dP, n=n, ld=n, block=128, stream=torch.cuda.current_stream())
        st = fw.fw_last_stats()
        if r:
            ms.append(st.solve_ms)
    fw.fw_free()
    m = statistics.median(ms)
    print(json.dumps({"config": a.config, "n": n, "opts": opts, "solve_ms": m, "min_ms": min(ms),
                      "tflops": 2 * n ** 3 / (m * 1e-3) / 1e12, "persistent": st.persistent, "phase1_ms": st.phase1_ms, "phase2_ms": st.phase2_ms, "rounds": st.rounds,
                      "p_method": st.p_method, "phase3_ms": st.phase3_ms, "post_ms": st.post_ms,
                      "launches": st.kernel_launches}), flush=True)

"""Run one device-resident solve of a BASELINE config (for ncu / sanitizer captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import apsp_inputs as gen  # noqa: E402
import paper_1811_01201_b200 as fw  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--block", type=int, default=0)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--nopath", action="store_true")
a = ap.parse_args()
c = dict(gen.CONFIGS[a.config])
if a.n:
    c["n"] = a.n
W = gen.generate(c["kind"], c["n"], c["seed"], p=c.get("p", 1.0), lo=c.get("lo", 1), hi=c.get("hi", 100))
dD = torch.from_numpy(W).cuda()
dP = None if a.nopath else torch.empty(W.shape, dtype=torch.int32, device="cuda")
fw.fw_init(0, fw.FW_TIMING)
f = fw.fw_solve_device_i32 if W.dtype.name == "int32" else fw.fw_solve_device_f32
for _ in range(a.reps):
    dD.copy_(torch.from_numpy(W).cuda())
    f(dD, dP, block=a.block or c["block"], stream=torch.cuda.current_stream())
    s = fw.fw_last_stats()
    print({k: round(v, 3) if isinstance(v, float) else v for k, v in s.as_dict().items()}, flush=True)
fw.fw_free()

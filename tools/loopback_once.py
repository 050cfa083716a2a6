"""One loopback-transport solve (every rank of a W-way block-row partition on this GPU) of a
BASELINE config, for ncu launch lists of the multi-GPU phase launches."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import apsp_inputs as gen  # noqa: E402
import paper_1811_01201_b200 as fw  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--world", type=int, default=8)
a = ap.parse_args()
c = gen.CONFIGS[a.config]
dW = gen.generate_torch(c["kind"], c["n"], c["seed"], device="cuda", p=c.get("p", 1.0), lo=c.get("lo", 1),
                        hi=c.get("hi", 100))
dP = torch.empty(dW.shape, dtype=torch.int32, device="cuda")
fw.fw_init(0, 0)
fw.fw_dist_loopback_solve_device_f32(dW, dP, block=c["block"], world=a.world, stream=torch.cuda.current_stream())
torch.cuda.synchronize()
fw.fw_free()
print("ok")

"""Host-entry pipeline probe: fw_solve with pinned host buffers at several chunk sizes
(0 = pipeline off); prints wall ms and the library's stats per run."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import apsp_inputs as gen  # noqa: E402
import paper_1811_01201_b200 as fw  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--chunks", default="0,8,16,32")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--pageable", action="store_true", help="NumPy-backed (pageable) host buffers")
a = ap.parse_args()
c = gen.CONFIGS[a.config]
dW = gen.generate_torch(c["kind"], c["n"], c["seed"], device="cuda", p=c.get("p", 1.0),
                        lo=c.get("lo", 1), hi=c.get("hi", 100))
hin = dW.cpu() if a.pageable else dW.cpu().pin_memory()
del dW
hD = torch.empty_like(hin) if a.pageable else torch.empty_like(hin).pin_memory()
hP = torch.empty(hin.shape, dtype=torch.int32)
if not a.pageable:
    hP = hP.pin_memory()
n = c["n"]
fw.fw_init(0, 0)
f = fw.fw_solve_i32 if hin.dtype == torch.int32 else fw.fw_solve
for ct in [int(x) for x in a.chunks.split(",")]:
    fw.fw_set_host_pipeline(ct)
    for r in range(a.reps + 1):
        hD.copy_(hin)
        t0 = time.perf_counter()
        f(hD, hP, block=c["block"])
        dt = (time.perf_counter() - t0) * 1e3
        s = fw.fw_last_stats()
        if r:
            print(f"{'pageable' if a.pageable else 'pinned'} chunk_tiles={ct} wall_ms={dt:.2f} gflops={2 * n ** 3 / dt / 1e6:.0f} "
                  f"lib_ms={s.solve_ms:.2f} chunks={s.host_chunks} h2d_exposed={s.h2d_ms:.2f} "
                  f"d2h_exposed={s.d2h_ms:.2f} launches={s.kernel_launches}", flush=True)
fw.fw_free()

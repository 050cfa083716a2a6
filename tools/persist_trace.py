"""Summarise a persistent-kernel item trace (FW_PERSIST_TRACE=path, one-GPU solve).

python tools/persist_trace.py trace.bin --n 4096
Each item has {taken, operands ready, done} (%globaltimer ns) and its CTA. Prints where the
CTA-time of the launch went: computing items, waiting for their operands (dependency polls), and
idle between items / at the tail; per item type; the per-round pivot chain (P1(K) done -> P1(K+1)
done); and the number of CTAs computing over time (ramp, steady state, tail)."""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_01201_b200 as fw  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("path")
ap.add_argument("--n", type=int, required=True)
ap.add_argument("--bins", type=int, default=40)
a = ap.parse_args()
raw = np.fromfile(a.path, dtype=np.int64)
magic, T, W, total, quarters, gap, grid, self_ = raw[:8]
assert magic == 0x46575453 and W == 1, "one-GPU traces only"
allrec = raw[8:].reshape(-1, 8).astype(np.uint64)
rec = allrec[:total]
lone = allrec[total:total + T]                  # the dedicated P1 CTA's records (if it ran)
items = list(fw.fw_persist_schedule(a.n, 1, {0: -2, 1: -3, 2: -4}[int(quarters)], int(gap)))
if (lone[:, 2] > 0).any():                      # its P1 items, appended as items of type P1
    for K in range(T):
        items.append((1 << 27) | (K << 18) | (K << 9) | K)
    rec = np.concatenate([rec[:len(items) - T], lone])
m = min(len(items), len(rec))
rec = rec[:m]
ok = rec[:, 2] > 0
t0 = rec[:, 0].astype(np.float64)
base = t0[ok].min()
t0 = (t0 - base) / 1e3                          # us
t1 = (rec[:, 1].astype(np.float64) - base) / 1e3
t2 = (rec[:, 2].astype(np.float64) - base) / 1e3
cta = (rec[:, 3] & 0xffffffff).astype(np.int64)
it = np.asarray(items[:m], dtype=np.uint64)
typ = ((it >> 27) & 3).astype(int)
K = ((it >> 18) & 511).astype(int)
span = t2[ok].max()
busy = (t2 - t0)[ok].sum()
wait = (t1 - t0)[ok].sum()
cap = float(grid) * span
out = {"T": int(T), "grid": int(grid), "items": int(ok.sum()), "quarters": int(quarters), "gap": int(gap),
       "makespan_us": span,
       "cta_time_fraction": {"computing": (busy - wait) / cap, "waiting_for_operands": wait / cap,
                             "idle_between_items_or_tail": 1 - busy / cap}}
names = {1: "P1", 2: "tile", 3: "quarter"}
per = {}
for t in (1, 2, 3):
    s = ok & (typ == t)
    if s.any():
        per[names[t]] = {"count": int(s.sum()), "mean_compute_us": float((t2 - t1)[s].mean()),
                         "mean_wait_us": float((t1 - t0)[s].mean()), "max_wait_us": float((t1 - t0)[s].max())}
out["per_type"] = per
# the steps between taking a tile and starting it (thread 0's clock): decode (incl. the next
# index's atomic), the barrier after it, the dependency polls, the barrier after them
ta = (rec[:, 4].astype(np.float64) - base) / 1e3
tb = (rec[:, 5].astype(np.float64) - base) / 1e3
tc = (rec[:, 6].astype(np.float64) - base) / 1e3
s = ok & (typ == 2)
out["tile_take_to_start_us"] = {"decode_and_atomic": float((ta - t0)[s].mean()), "barrier1": float((tb - ta)[s].mean()),
                                "polls": float((tc - tb)[s].mean()), "barrier2": float((t1 - tc)[s].mean())}
p1 = ok & (typ == 1)
p1_done = np.sort(t2[p1])
out["p1_done_interval_us"] = {"mean": float(np.diff(p1_done).mean()) if len(p1_done) > 1 else None,
                              "max": float(np.diff(p1_done).max()) if len(p1_done) > 1 else None}
# CTAs computing over time
edges = np.linspace(0, span, a.bins + 1)
conc = []
for lo, hi in zip(edges[:-1], edges[1:]):
    ov = np.clip(np.minimum(t2[ok], hi) - np.maximum(t1[ok], lo), 0, None).sum()
    conc.append(round(float(ov / (hi - lo)), 1))
out["ctas_computing_per_bin"] = conc
# per-CTA idle: gaps between consecutive items of one CTA
gaps = []
for c in np.unique(cta[ok]):
    s = np.where(ok & (cta == c))[0]
    s = s[np.argsort(t0[s])]
    if len(s) > 1:
        gaps.append((t0[s[1:]] - t2[s[:-1]]).clip(0).sum())
out["mean_idle_between_items_us_per_cta"] = float(np.mean(gaps)) if gaps else 0.0
print(json.dumps(out, indent=1))

"""Shared helpers for the GPU parity tests (test side only)."""
from __future__ import annotations

import numpy as np

import apsp_inputs as gen
import oracle

INF = gen.INF_I32


def exact_data(W: np.ndarray) -> bool:
    """Integer-valued data (INT32, or FP32 holding integers): D must be bit-exact."""
    if W.dtype == np.int32:
        return True
    fin = W[np.isfinite(W)]
    return bool(np.all(fin == np.round(fin)))


def assert_D_matches(D: np.ndarray, Dref: np.ndarray, exact: bool, rtol: float = 1e-5):
    """BJ:5: bit-exact for integer data; rel 1e-5 for real FP32; INF must match exactly."""
    if exact:
        if not np.array_equal(D, Dref):
            bad = np.argwhere(D != Dref)
            i, j = bad[0]
            raise AssertionError(f"{len(bad)} mismatches, first ({i},{j}): got {D[i, j]} want {Dref[i, j]}")
        return
    Dd = D.astype(np.float64)
    Rd = Dref.astype(np.float64)
    inf_d, inf_r = np.isinf(Dd), np.isinf(Rd)
    assert np.array_equal(inf_d, inf_r), "INF pattern differs"
    fin = ~inf_r
    rel = np.abs(Dd[fin] - Rd[fin]) / np.maximum(1.0, np.abs(Rd[fin]))
    assert rel.max(initial=0.0) <= rtol, f"max rel err {rel.max()}"


def next_consistency(W: np.ndarray, D: np.ndarray, nxt: np.ndarray, exact: bool, rtol=1e-5,
                     rows=None, chunk=1024) -> int:
    """O(n^2) local check of a next-hop matrix (SURVEY.md §4 suite 7): for every reachable
    i != j, h = next[i][j] is an edge of W and W[i][h] + D[h][j] == D[i][j] (exact for
    integer data, rel rtol for reals); next[i][i] == i; unreachable -> -1. Returns #bad."""
    n = W.shape[0]

    def f64(a):   # gathered values only: the full matrices may be 4 GiB (C5)
        out = a.astype(np.float64)
        if W.dtype == np.int32:
            out[a >= INF] = np.inf
        return out
    rows = np.arange(n) if rows is None else np.asarray(rows)
    bad = 0
    for s in range(0, len(rows), chunk):
        r = rows[s:s + chunk]
        h = nxt[r]
        d = f64(D[r])
        reach = np.isfinite(d)
        diag = (r[:, None] == np.arange(n)[None, :])
        bad += int(np.sum(diag & (h != r[:, None])))
        bad += int(np.sum(~reach & (h != -1)))
        m = reach & ~diag
        hh = np.where(m, h, 0)
        ok_range = (hh >= 0) & (hh < n)
        bad += int(np.sum(m & ~ok_range))
        hh = np.clip(hh, 0, n - 1)
        w = f64(W[r[:, None], hh])
        dh = f64(D[hh, np.arange(n)[None, :]])
        lhs = w + dh
        if exact:
            good = lhs == d
        else:
            good = np.abs(lhs - d) <= rtol * np.maximum(1.0, np.abs(d))
        bad += int(np.sum(m & ~(good & np.isfinite(w))))
    return bad

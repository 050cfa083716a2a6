"""Seeded synthetic inputs for the blocked Floyd-Warshall APSP path.

This module is shared by the oracle side (``oracle/``, ``tests/``) and the
product side (``bench.py``). It holds NONE of the method's arithmetic: it only
draws adjacency matrices W (the paper's initial distance matrix D, PAPER.md
§3 "D_{i,j} is initialized with the original distance from node i to node j")
from a counter-based generator, so that every consumer gets bit-identical
inputs for (config, seed).

Generator (SURVEY.md §8(d) "Counter-based generator")::

    z(seed, stream, i, j) = splitmix64_fin(seed*G ^ stream*H ^ (i*n + j))
    int weight  in [lo,hi] : lo + ((z>>32) * (hi-lo+1)) >> 32         (stream 0)
    real weight in [1,100) : float32(1 + 99 * (z>>40) * 2^-24)          (stream 0)
    ER edge present        : (z1>>11) * 2^-53 < p,  z1 = z(seed,1,i,j)
    sources                : first distinct z(seed,7,0,t) % n, sorted

The paper states no generator (§5.1 only names N and "different
workloads"); the recipe and each config's shape follow BASELINE.json configs
(see DESIGN.md "Input recipe").
"""
from __future__ import annotations

import numpy as np

INF_I32 = 0x3FFFFFFF          # INT32 sentinel, INT32_MAX/2 (BASELINE.json configs[2])
INF_F32 = np.float32(np.inf)  # FP32 sentinel: IEEE +inf

_G = np.uint64(0x9E3779B97F4A7C15)
_H = np.uint64(0xD1B54A32D192ED03)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64_fin(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    x = x + _G
    x = (x ^ (x >> np.uint64(30))) * _M1
    x = (x ^ (x >> np.uint64(27))) * _M2
    return x ^ (x >> np.uint64(31))


def counter(seed: int, stream: int, n: int, rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
    """z(seed, stream, i, j) for the outer product rows x cols (uint64)."""
    with np.errstate(over="ignore"):
        base = np.uint64(seed) * _G ^ np.uint64(stream) * _H
        idx = (rows.astype(np.uint64)[:, None] * np.uint64(n)) + cols.astype(np.uint64)[None, :]
        return splitmix64_fin(base ^ idx)


def _int_weights(z: np.ndarray, lo: int, hi: int) -> np.ndarray:
    span = np.uint64(hi - lo + 1)
    with np.errstate(over="ignore"):
        return (np.uint64(lo) + (((z >> np.uint64(32)) * span) >> np.uint64(32))).astype(np.int64)


def _real_weights(z: np.ndarray) -> np.ndarray:
    u = (z >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)
    return (1.0 + 99.0 * u).astype(np.float32)


def generate(kind: str, n: int, seed: int, p: float = 1.0, lo: int = 1, hi: int = 100,
             chunk_rows: int = 512, rows: tuple[int, int] | None = None) -> np.ndarray:
    """Adjacency matrix W (n x n, row-major, C-contiguous) for one workload kind.

    kind:
      "complete_int"  FP32 holding integers uniform in [lo,hi]  (configs[0], configs[3])
      "complete_real" FP32 uniform real in [1,100)               (configs[1], configs[4])
      "er_int"        INT32 integers in [lo,hi] with prob p, else INF_I32   (configs[2])
      "er_int_f32"    FP32 integers in [lo,hi] with prob p, else +inf
      "er_real"       FP32 real in [1,100) with prob p, else +inf
    The diagonal is 0 in every kind. rows=(r0, r1) draws only rows [r0, r1) of the same
    matrix (a multi-GPU rank's block-rows).
    """
    if n <= 0:
        raise ValueError("n must be positive")
    dtype = np.int32 if kind == "er_int" else np.float32
    lo_row, hi_row = (0, n) if rows is None else (max(0, rows[0]), min(n, rows[1]))
    W = np.empty((max(0, hi_row - lo_row), n), dtype=dtype)
    cols = np.arange(n, dtype=np.int64)
    for r0 in range(lo_row, hi_row, chunk_rows):
        rows = np.arange(r0, min(hi_row, r0 + chunk_rows), dtype=np.int64)
        z0 = counter(seed, 0, n, rows, cols)
        if kind in ("complete_int", "er_int", "er_int_f32"):
            w = _int_weights(z0, lo, hi)
        elif kind in ("complete_real", "er_real"):
            w = _real_weights(z0)
        else:
            raise ValueError(f"unknown kind {kind!r}")
        del z0
        if kind.startswith("er_"):
            z1 = counter(seed, 1, n, rows, cols)
            present = (z1 >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) < p
            del z1
            inf = INF_I32 if dtype == np.int32 else np.inf
            w = np.where(present, w, inf)
        blk = W[rows[0] - lo_row:rows[-1] + 1 - lo_row]
        blk[...] = w.astype(dtype)
        blk[np.arange(len(rows)), rows] = 0
    return W


def _s64(c: int) -> int:
    """uint64 constant as the int64 with the same bits (torch has no full uint64 arithmetic)."""
    return c - (1 << 64) if c >= (1 << 63) else c


def generate_torch(kind: str, n: int, seed: int, device="cpu", p: float = 1.0, lo: int = 1,
                   hi: int = 100, rows: tuple[int, int] | None = None, chunk_rows: int = 1024):
    """The same matrix as generate(), drawn with torch int64 ops (wrapping multiply, logical
    shifts emulated by masking) so large inputs can be created directly in device memory
    (bench.py at n >= 32768). Bit-identical to generate() (tests/test_oracle.py pins it)."""
    import torch
    if n <= 0:
        raise ValueError("n must be positive")
    is_int = kind == "er_int"
    dtype = torch.int32 if is_int else torch.float32
    lo_row, hi_row = (0, n) if rows is None else (max(0, rows[0]), min(n, rows[1]))
    W = torch.empty((max(0, hi_row - lo_row), n), dtype=dtype, device=device)
    G, M1, M2, H = (_s64(int(c)) for c in (_G, _M1, _M2, _H))

    def shr(x, s):                       # logical right shift of the 64-bit pattern
        return (x >> s) & ((1 << (64 - s)) - 1)

    def fin(x):
        x = x + G
        x = (x ^ shr(x, 30)) * M1
        x = (x ^ shr(x, 27)) * M2
        return x ^ shr(x, 31)

    def z_of(stream, r):
        base = _s64((seed * int(_G)) % (1 << 64) ^ (stream * int(_H)) % (1 << 64))
        idx = r[:, None] * n + torch.arange(n, dtype=torch.int64, device=device)[None, :]
        return fin(base ^ idx)

    for r0 in range(lo_row, hi_row, chunk_rows):
        r = torch.arange(r0, min(hi_row, r0 + chunk_rows), dtype=torch.int64, device=device)
        z0 = z_of(0, r)
        if kind in ("complete_int", "er_int", "er_int_f32"):
            w = lo + ((shr(z0, 32) * (hi - lo + 1)) >> 32)
        elif kind in ("complete_real", "er_real"):
            w = (1.0 + 99.0 * (shr(z0, 40).to(torch.float64) * (2.0 ** -24))).to(torch.float32)
        else:
            raise ValueError(f"unknown kind {kind!r}")
        del z0
        if kind.startswith("er_"):
            z1 = z_of(1, r)
            present = shr(z1, 11).to(torch.float64) * (2.0 ** -53) < p
            del z1
            w = torch.where(present, w, INF_I32 if is_int else float("inf"))
        blk = W[r0 - lo_row:r0 - lo_row + len(r)]
        blk.copy_(w.to(dtype))
        blk[torch.arange(len(r), device=device), r] = 0
    return W


def sources(n: int, seed: int, count: int = 64) -> np.ndarray:
    """`count` distinct seeded source vertices (sorted), SURVEY.md C-16."""
    count = min(count, n)
    out: list[int] = []
    seen = set()
    t = 0
    while len(out) < count:
        ts = np.arange(t, t + 4 * count, dtype=np.int64)
        z = counter(seed, 7, 1, np.zeros(1, dtype=np.int64), ts)[0]
        for v in (z % np.uint64(n)).tolist():
            if v not in seen:
                seen.add(v)
                out.append(int(v))
                if len(out) == count:
                    break
        t += 4 * count
    return np.array(sorted(out), dtype=np.int64)


# ---- structured inputs with closed-form answers (used as pins) ----

def ring(n: int, w: int = 1, dtype=np.float32) -> np.ndarray:
    """Directed ring i -> i+1 (mod n) with weight w; all other pairs INF."""
    inf = INF_I32 if dtype == np.int32 else np.inf
    W = np.full((n, n), inf, dtype=dtype)
    idx = np.arange(n)
    W[idx, (idx + 1) % n] = w
    W[idx, idx] = 0
    return W


def ring_with_chords(n: int, seed: int, chords: int, dtype=np.float32) -> np.ndarray:
    """Ring of weight 1 plus `chords` random chords u->v of weight n (never shortcuts)."""
    W = ring(n, 1, dtype)
    if n < 3:
        return W
    z = counter(seed, 5, n, np.arange(1, dtype=np.int64), np.arange(2 * chords, dtype=np.int64))[0]
    uv = (z % np.uint64(n)).astype(np.int64).reshape(-1, 2)
    for u, v in uv:
        if u != v and (v - u) % n != 1:
            W[u, v] = n
    return W


def abs_diff(n: int, dtype=np.float32) -> np.ndarray:
    """Complete graph with w(i,j) = |i-j| (direct edges optimal, massive ties)."""
    idx = np.arange(n)
    return np.abs(idx[:, None] - idx[None, :]).astype(dtype)


def uniform_complete(n: int, c: float, dtype=np.float32) -> np.ndarray:
    W = np.full((n, n), c, dtype=dtype)
    np.fill_diagonal(W, 0)
    return W


def empty_graph(n: int, dtype=np.float32) -> np.ndarray:
    inf = INF_I32 if dtype == np.int32 else np.inf
    W = np.full((n, n), inf, dtype=dtype)
    np.fill_diagonal(W, 0)
    return W


def two_components(n: int, seed: int, p: float = 0.05, dtype=np.int32) -> np.ndarray:
    """ER graph restricted to two halves with no edges between them (INF across)."""
    kind = "er_int" if dtype == np.int32 else "er_int_f32"
    W = generate(kind, n, seed, p=p, lo=1, hi=1000)
    h = n // 2
    inf = INF_I32 if dtype == np.int32 else np.inf
    W[:h, h:] = inf
    W[h:, :h] = inf
    return W


# BASELINE.json configs (index = configs[i]); SURVEY.md §8(d) table.
CONFIGS = {
    "C1": dict(kind="complete_int", n=512, seed=1, block=32, dtype="f32", exact=True),
    "C2": dict(kind="complete_real", n=4096, seed=2, block=128, dtype="f32", exact=False),
    "C3": dict(kind="er_int", n=8192, seed=3, block=128, dtype="i32", exact=True, p=0.1, lo=1, hi=1000),
    "C4": dict(kind="complete_int", n=16384, seed=4, block=128, dtype="f32", exact=True),
    "C5": dict(kind="complete_real", n=32768, seed=5, block=128, dtype="f32", exact=False),
}


def config_matrix(name: str, rows: tuple[int, int] | None = None) -> np.ndarray:
    c = CONFIGS[name]
    return generate(c["kind"], c["n"], c["seed"], p=c.get("p", 1.0), lo=c.get("lo", 1), hi=c.get("hi", 100),
                    rows=rows)

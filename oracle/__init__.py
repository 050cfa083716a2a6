"""CPU oracle for the blocked Floyd–Warshall APSP hot path (arxiv 1811.01201).

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package. It shares no code with ``paper_1811_01201_b200`` (the product) and the
product never imports it.

Every routine is a thin ctypes marshaller around ``fw_oracle.c`` (plain C, fp32
without fast-math / contraction for the FW triple loop, double / int64 for the
independent checkers). See the C file header for the paper citations.

Parity pins (what the oracle itself is checked against, tests/test_oracle.py):
  * Dijkstra from every source (independent algorithm), brute-force simple-path
    enumeration (n <= 8), repeated min-plus squaring (n <= 64), scipy.sparse.csgraph
    (third-party), closed forms (ring, |i-j|, uniform complete graph), SPEC.md worked
    examples (tests/golden/), and invariants (diag 0, triangle inequality,
    idempotence, transpose / permutation / scaling covariance).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "fw_oracle.c")

INF_I32 = 0x3FFFFFFF
MODE_NEXT = 0
MODE_LASTK = 1

CFLAGS = ["-O3", "-march=x86-64-v3", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
          "-fPIC", "-shared", "-Wall"]


def build(force: bool = False) -> str:
    """Compile fw_oracle.c into liboracle.so (gcc)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        L.oracle_fw_f32.argtypes = [P, P, I64, ctypes.c_int]
        L.oracle_fw_i32.argtypes = [P, P, I64, ctypes.c_int]
        L.oracle_fw_f32_steps.argtypes = [P, P, I64, I64, I64]
        L.oracle_dijkstra_f32.argtypes = [P, I64, P, I64, P]
        L.oracle_dijkstra_i32.argtypes = [P, I64, P, I64, P]
        L.oracle_bruteforce_f64.argtypes = [P, I64, P]
        L.oracle_minplus_closure_f64.argtypes = [P, I64, P]
        for f in (L.oracle_check_next, L.oracle_check_lastk):
            f.argtypes = [P, P, P, I64, P, I64, ctypes.c_double, P]
            f.restype = I64
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def fw(W: np.ndarray, path: str | None = "next"):
    """Naive triple-loop Floyd–Warshall (paper Fig. 1).

    W: n x n float32 (+inf = no edge) or int32 (INF_I32 = no edge). Returns (D, P)
    with P = None if path is None, next-hop matrix if "next", the paper's last
    intermediate node if "lastk". Diagonal forced to 0. Strict '<'.
    """
    W = np.asarray(W)
    n = W.shape[0]
    assert W.shape == (n, n)
    D = np.ascontiguousarray(W).copy()
    P = None if path is None else np.empty((n, n), dtype=np.int32)
    mode = MODE_LASTK if path == "lastk" else MODE_NEXT
    if D.dtype == np.float32:
        rc = lib().oracle_fw_f32(_ptr(D), _ptr(P) if P is not None else None, n, mode)
    elif D.dtype == np.int32:
        rc = lib().oracle_fw_i32(_ptr(D), _ptr(P) if P is not None else None, n, mode)
    else:
        raise TypeError(f"unsupported dtype {D.dtype}")
    assert rc == 0
    return D, P


def fw_steps(D: np.ndarray, P: np.ndarray | None, k0: int, k1: int) -> None:
    """Outer iterations k in [k0, k1) of the FP32 triple loop, in place (timing samples)."""
    assert D.dtype == np.float32 and D.flags["C_CONTIGUOUS"]
    n = D.shape[0]
    rc = lib().oracle_fw_f32_steps(_ptr(D), _ptr(P) if P is not None else None, n, k0, k1)
    assert rc == 0


def dijkstra(W: np.ndarray, srcs) -> np.ndarray:
    """Exact distances from each source in `srcs` (rows), by dense Dijkstra.

    float32 W -> float64 result (+inf unreachable); int32 W -> int64 result with
    unreachable mapped to INF_I32 (the output sentinel of the APSP result).
    """
    W = np.ascontiguousarray(W)
    n = W.shape[0]
    s = np.ascontiguousarray(np.asarray(srcs, dtype=np.int64))
    if W.dtype == np.float32:
        out = np.empty((len(s), n), dtype=np.float64)
        rc = lib().oracle_dijkstra_f32(_ptr(W), n, _ptr(s), len(s), _ptr(out))
    elif W.dtype == np.int32:
        out = np.empty((len(s), n), dtype=np.int64)
        rc = lib().oracle_dijkstra_i32(_ptr(W), n, _ptr(s), len(s), _ptr(out))
        out[out == np.iinfo(np.int64).max] = INF_I32
    else:
        raise TypeError(W.dtype)
    assert rc == 0
    return out


def _as_f64(W: np.ndarray) -> np.ndarray:
    Wd = np.asarray(W).astype(np.float64)
    if np.asarray(W).dtype == np.int32:
        Wd[np.asarray(W) >= INF_I32] = np.inf
    return np.ascontiguousarray(Wd)


def bruteforce(W: np.ndarray) -> np.ndarray:
    """All-pairs minimum over simple paths by exhaustive DFS (n <= 8), float64."""
    Wd = _as_f64(W)
    n = Wd.shape[0]
    assert n <= 8
    out = np.empty_like(Wd)
    assert lib().oracle_bruteforce_f64(_ptr(Wd), n, _ptr(out)) == 0
    return out


def minplus_closure(W: np.ndarray) -> np.ndarray:
    """Repeated min-plus squaring, float64, n <= 64 recommended."""
    Wd = _as_f64(W)
    n = Wd.shape[0]
    out = np.empty_like(Wd)
    assert lib().oracle_minplus_closure_f64(_ptr(Wd), n, _ptr(out)) == 0
    return out


def check_paths(W: np.ndarray, D: np.ndarray, P: np.ndarray, rows=None, rtol: float = 0.0,
                mode: str = "next"):
    """Count pairs whose reconstructed path is invalid (see fw_oracle.c).

    Returns (n_bad, first_bad_flat_index or -1).
    """
    Wd = _as_f64(W)
    Dd = _as_f64(D)
    n = Wd.shape[0]
    P = np.ascontiguousarray(P, dtype=np.int32)
    rows = np.arange(n, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    first = np.array([-1], dtype=np.int64)
    f = lib().oracle_check_next if mode == "next" else lib().oracle_check_lastk
    bad = f(_ptr(Wd), _ptr(Dd), _ptr(P), n, _ptr(rows), len(rows), float(rtol), _ptr(first))
    return int(bad), int(first[0])

"""Pins for the CPU oracle (oracle/): everything here is checked against something
other than the oracle itself — an independent algorithm (Dijkstra, brute force,
min-plus squaring), a third-party library (scipy.sparse.csgraph), closed forms,
SPEC.md worked examples (tests/golden/), or mathematical invariants.
SURVEY.md §8(c) "What pins each part".
"""
import numpy as np
import pytest

import apsp_inputs as gen
import oracle
from conftest import golden_names, load_golden

INF = gen.INF_I32


def rand_graph(n, seed, p=0.5, lo=1, hi=20, dtype=np.float32):
    kind = "er_int" if dtype == np.int32 else "er_int_f32"
    return gen.generate(kind, n, seed, p=p, lo=lo, hi=hi)


def as_f64(W):
    Wd = W.astype(np.float64)
    if W.dtype == np.int32:
        Wd[W >= INF] = np.inf
    return Wd


# ---------------------------------------------------------------- golden (SPEC examples)
@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("dtype", [np.float32, np.int32])
def test_golden(name, dtype):
    g = load_golden(name)
    W = g["W"]
    if dtype == np.int32:
        Wi = np.where(np.isinf(W), INF, W).astype(np.int32)
        D, P = oracle.fw(Wi, "next")
        Dexp = np.where(np.isinf(g["D"]), INF, g["D"]).astype(np.int32)
    else:
        D, P = oracle.fw(W.astype(np.float32), "next")
        Dexp = g["D"].astype(np.float32)
    np.testing.assert_array_equal(D, Dexp)
    if "NEXT" in g:
        np.testing.assert_array_equal(P, g["NEXT"])
    if "LASTK" in g:
        # both branches of the oracle's LAST_K mode (oracle_fw_f32 / oracle_fw_i32 mode 1)
        Wl = Wi if dtype == np.int32 else W.astype(np.float32)
        DL, PL = oracle.fw(Wl, "lastk")
        np.testing.assert_array_equal(DL, Dexp)
        np.testing.assert_array_equal(PL, g["LASTK"])


# ------------------------------------------------------------- independent algorithms
@pytest.mark.parametrize("seed", range(40))
def test_vs_bruteforce_tiny(seed):
    n = 2 + seed % 7   # 2..8
    W = rand_graph(n, seed, p=0.45, hi=9)
    D, P = oracle.fw(W)
    B = oracle.bruteforce(W)
    np.testing.assert_array_equal(D.astype(np.float64), B)
    assert oracle.check_paths(W, D, P)[0] == 0
    Wi = np.where(np.isinf(W), INF, W).astype(np.int32)
    Di, _ = oracle.fw(Wi)
    np.testing.assert_array_equal(as_f64(Di), B)


@pytest.mark.parametrize("seed", range(12))
def test_vs_minplus_squaring(seed):
    n = [16, 33, 64][seed % 3]
    W = rand_graph(n, 100 + seed, p=0.15 + 0.05 * (seed % 4), hi=50)
    D, _ = oracle.fw(W)
    np.testing.assert_array_equal(D.astype(np.float64), oracle.minplus_closure(W))


@pytest.mark.parametrize("kind,n,p", [("complete_int", 256, 1.0), ("er_int", 300, 0.02),
                                      ("er_int", 257, 0.1), ("er_int_f32", 200, 0.01)])
def test_vs_dijkstra_all_sources(kind, n, p):
    W = gen.generate(kind, n, 7, p=p, lo=1, hi=1000 if kind.startswith("er") else 100)
    D, P = oracle.fw(W)
    R = oracle.dijkstra(W, np.arange(n))
    if W.dtype == np.int32:
        np.testing.assert_array_equal(D.astype(np.int64), R)
    else:
        np.testing.assert_array_equal(D.astype(np.float64), R)
    assert oracle.check_paths(W, D, P)[0] == 0
    # LAST_K branch of the same type (INT32: oracle_fw_i32 mode 1): same D, and every path
    # expanded recursively from P sums to D over the original edges
    DL, PL = oracle.fw(W, "lastk")
    np.testing.assert_array_equal(DL, D)
    assert oracle.check_paths(W, DL, PL, mode="lastk")[0] == 0
    # -1 exactly where no intermediate vertex improved: the direct edge is optimal or no path
    direct = (W == D) | (D >= INF if W.dtype == np.int32 else np.isinf(D))
    assert np.all(PL[~direct] >= 0)


def test_real_weights_within_tolerance_of_exact():
    """FP32 triple loop vs exact (double) Dijkstra: within rel 1e-5 (BJ:5)."""
    n = 384
    W = gen.generate("complete_real", n, 2)
    D, P = oracle.fw(W)
    R = oracle.dijkstra(W, np.arange(n))
    rel = np.abs(D.astype(np.float64) - R) / np.maximum(1.0, np.abs(R))
    assert rel.max() < 1e-5
    assert oracle.check_paths(W, D, P, rtol=1e-5)[0] == 0
    _, PL = oracle.fw(W, "lastk")
    assert oracle.check_paths(W, D, PL, rtol=1e-5, mode="lastk")[0] == 0


def test_vs_scipy():
    from scipy.sparse.csgraph import csgraph_from_dense, shortest_path
    n = 200
    W = gen.generate("er_int_f32", n, 11, p=0.03, lo=1, hi=1000)
    D, _ = oracle.fw(W)
    G = csgraph_from_dense(W.astype(np.float64), null_value=np.inf)
    S = shortest_path(G, method="D", directed=True)
    np.testing.assert_array_equal(D.astype(np.float64), S)


# ------------------------------------------------------------------------ closed forms
@pytest.mark.parametrize("n", [1, 2, 5, 64, 129])
def test_ring_closed_form(n):
    W = gen.ring(n, 1)
    D, P = oracle.fw(W)
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    np.testing.assert_array_equal(D, ((j - i) % n).astype(np.float32))
    nxt = np.where(i == j, i, (i + 1) % n)
    np.testing.assert_array_equal(P, nxt)


@pytest.mark.parametrize("n", [3, 50, 128])
def test_abs_diff_closed_form(n):
    W = gen.abs_diff(n)
    D, P = oracle.fw(W)
    np.testing.assert_array_equal(D, W)      # direct edge optimal (ties everywhere)
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    np.testing.assert_array_equal(P, j)      # strict '<' never replaces a direct edge


def test_ring_with_chords_and_uniform():
    n = 97
    W = gen.ring_with_chords(n, 3, 300)
    D, P = oracle.fw(W)
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    np.testing.assert_array_equal(D, ((j - i) % n).astype(np.float32))
    assert oracle.check_paths(W, D, P)[0] == 0
    U = gen.uniform_complete(40, 7.0)
    DU, _ = oracle.fw(U)
    np.testing.assert_array_equal(DU, U)


def test_single_vertex_and_empty():
    D, P = oracle.fw(np.array([[5.0]], dtype=np.float32))
    assert D[0, 0] == 0 and P[0, 0] == 0            # diagonal forced to 0 (reading R4)
    E = gen.empty_graph(9, np.int32)
    D, P = oracle.fw(E)
    np.testing.assert_array_equal(D, E)
    assert (P[~np.eye(9, dtype=bool)] == -1).all()


# -------------------------------------------------------------------------- invariants
def test_invariants():
    n = 160
    W = gen.generate("er_int_f32", n, 21, p=0.05, lo=1, hi=100)
    D, P = oracle.fw(W)
    assert (np.diag(D) == 0).all()
    assert (D <= np.where(np.eye(n, dtype=bool), 0, W)).all()
    # triangle inequality: D[i][j] <= D[i][k] + D[k][j] for all i, j, k (exact ints)
    Dd = D.astype(np.float64)
    for k in range(n):
        assert (Dd <= Dd[:, [k]] + Dd[[k], :]).all()
    # idempotence
    D2, _ = oracle.fw(D)
    np.testing.assert_array_equal(D2, D)
    # transpose covariance: D(W^T) = D(W)^T
    DT, _ = oracle.fw(np.ascontiguousarray(W.T))
    np.testing.assert_array_equal(DT, D.T)
    # permutation covariance
    rng = np.random.default_rng(5)
    pi = rng.permutation(n)
    Dp, _ = oracle.fw(np.ascontiguousarray(W[np.ix_(pi, pi)]))
    np.testing.assert_array_equal(Dp, D[np.ix_(pi, pi)])
    # scaling: D(2W) = 2 D(W) (exact for integers)
    Ds, _ = oracle.fw((2 * W).astype(np.float32))
    np.testing.assert_array_equal(Ds, 2 * D)


def test_path_checker_detects_corruption():
    """The validator must fail on a corrupted P or D."""
    n = 64
    W = gen.generate("complete_int", n, 3)
    D, P = oracle.fw(W)
    assert oracle.check_paths(W, D, P)[0] == 0
    # find an improved pair (next != j) and corrupt it to the direct edge
    i, j = np.argwhere((P != np.arange(n)[None, :]) & ~np.eye(n, dtype=bool))[0]
    Pc = P.copy()
    Pc[i, j] = j
    bad, first = oracle.check_paths(W, D, Pc)
    assert bad >= 1 and first == i * n + j
    Dc = D.copy()
    Dc[3, 7] += 1
    assert oracle.check_paths(W, Dc, P)[0] >= 1
    _, PL = oracle.fw(W, "lastk")
    assert oracle.check_paths(W, D, PL, mode="lastk")[0] == 0
    PL2 = PL.copy()
    PL2[i, j] = -1
    assert oracle.check_paths(W, D, PL2, mode="lastk")[0] >= 1


def test_int32_extremes():
    """INT32 sentinel arithmetic: INF + INF must not overflow (reading R3)."""
    n = 5
    W = np.full((n, n), INF, dtype=np.int32)
    W[0, 1] = 1_000_000
    W[1, 2] = 2_000_000
    D, P = oracle.fw(W)
    assert D[0, 2] == 3_000_000 and P[0, 2] == 1
    assert D[2, 0] == INF and P[2, 0] == -1


# --------------------------------------------------------------------------- generator
def test_generator_determinism_and_ranges():
    a = gen.generate("complete_int", 300, 9)
    b = gen.generate("complete_int", 300, 9)
    np.testing.assert_array_equal(a, b)
    off = a[~np.eye(300, dtype=bool)]
    assert off.min() == 1 and off.max() == 100 and (off == np.round(off)).all()
    r = gen.generate("complete_real", 300, 9)
    off = r[~np.eye(300, dtype=bool)]
    assert off.min() >= 1.0 and off.max() < 100.0
    assert (np.diag(a) == 0).all() and (np.diag(r) == 0).all()
    # chunking does not change the stream
    np.testing.assert_array_equal(gen.generate("complete_real", 300, 9, chunk_rows=7), r)


def test_generator_er_density():
    n, p = 1000, 0.1
    W = gen.generate("er_int", n, 3, p=p, lo=1, hi=1000)
    m = n * (n - 1)
    edges = int((W[~np.eye(n, dtype=bool)] < INF).sum())
    sigma = np.sqrt(m * p * (1 - p))
    assert abs(edges - m * p) < 5 * sigma
    fin = W[(W < INF) & ~np.eye(n, dtype=bool)]
    assert fin.min() >= 1 and fin.max() <= 1000


def test_sources():
    s = gen.sources(16384, 4)
    assert len(s) == 64 and len(set(s.tolist())) == 64 and (np.diff(s) > 0).all()
    np.testing.assert_array_equal(s, gen.sources(16384, 4))
    assert len(gen.sources(10, 1)) == 10


def test_fw_steps_equals_full_loop():
    """The bounded-sample entry used for CPU timing runs the same loop as oracle.fw."""
    n = 96
    W = gen.generate("complete_real", n, 4)
    D, P = oracle.fw(W)
    D2 = W.copy()
    np.fill_diagonal(D2, 0)
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    P2 = np.where(i == j, i, np.where(np.isinf(D2), -1, j)).astype(np.int32)
    oracle.fw_steps(D2, P2, 0, 40)
    oracle.fw_steps(D2, P2, 40, n)
    np.testing.assert_array_equal(D, D2)
    np.testing.assert_array_equal(P, P2)


def test_generator_row_ranges():
    """A rank's rows drawn alone equal the same rows of the full matrix."""
    full = gen.generate("er_int", 700, 5, p=0.1, lo=1, hi=1000)
    part = gen.generate("er_int", 700, 5, p=0.1, lo=1, hi=1000, rows=(256, 512), chunk_rows=100)
    np.testing.assert_array_equal(part, full[256:512])
    assert gen.generate("complete_real", 300, 1, rows=(384, 512)).shape == (0, 300)

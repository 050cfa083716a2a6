"""fw_path (host-only path reconstruction) on P matrices
from the CPU oracle: next-hop and LAST_K forms, checked against the paper's definition of a
shortest path (consecutive vertices are edges of W, the weights sum to D[i][j], no vertex
repeats) and the SPEC worked example; no GPU needed."""
import ctypes

import numpy as np
import pytest

import apsp_inputs as gen
import oracle
from conftest import load_golden

fw = pytest.importorskip("paper_1811_01201_b200")


def edge_sum(W, path):
    w = W.astype(np.float64)
    if W.dtype == np.int32:
        w[W >= gen.INF_I32] = np.inf
    return sum(w[a, b] for a, b in zip(path, path[1:]))


def check_all_pairs(W, mode):
    path = "lastk" if mode == fw.FW_PATH_LAST_K else "next"
    D, P = oracle.fw(W, path)
    n = W.shape[0]
    Df = D.astype(np.float64)
    if W.dtype == np.int32:
        Df[D >= gen.INF_I32] = np.inf
    for i in range(n):
        for j in range(n):
            p = fw.fw_path(P, i, j, mode, dist=D)
            if not np.isfinite(Df[i, j]):
                assert p == [], (i, j, p)
                continue
            assert p[0] == i and p[-1] == j and len(set(p)) == len(p), (i, j, p)
            assert edge_sum(W, p) == Df[i, j], (i, j, p)


def test_spec_chain_example():
    """n = 3, d[0][2] = 3 through vertex 1."""
    g = load_golden("spec_n3_chain.txt")
    W = g["W"].astype(np.float32)
    for mode, path in ((fw.FW_PATH_NEXT_HOP, "next"), (fw.FW_PATH_LAST_K, "lastk")):
        D, P = oracle.fw(W, path)
        assert fw.fw_path(P, 0, 2, mode, dist=D) == [0, 1, 2]
        assert fw.fw_path(P, 1, 1, mode, dist=D) == [1]


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("seed", range(3))
def test_all_pairs_complete_and_sparse(mode, seed):
    check_all_pairs(gen.generate("complete_int", 48, 500 + seed), mode)
    check_all_pairs(gen.generate("er_int", 60, 510 + seed, p=0.05, lo=1, hi=40), mode)


@pytest.mark.parametrize("mode", [0, 1])
def test_ring_long_paths(mode):
    """Ring of 200: the i -> i-1 path has 199 hops (deep LAST_K expansion, no recursion)."""
    n = 200
    W = gen.ring(n, 3, dtype=np.int32)
    path = "lastk" if mode else "next"
    D, P = oracle.fw(W, path)
    p = fw.fw_path(P, 5, 4, mode, dist=D)
    assert p == [(5 + t) % n for t in range(n)]


def test_unreachable_without_dist_next_hop():
    W = gen.two_components(40, 3, dtype=np.int32)
    D, P = oracle.fw(W, "next")
    i, j = np.argwhere(D >= gen.INF_I32)[0]
    assert fw.fw_path(P, int(i), int(j), fw.FW_PATH_NEXT_HOP) == []


def test_errors():
    W = gen.generate("complete_int", 16, 7)
    D, P = oracle.fw(W, "next")
    with pytest.raises(fw.FwError) as e:
        fw.fw_path(P, 0, 16)
    assert e.value.code == fw.FW_EINVAL
    with pytest.raises(fw.FwError):
        fw.fw_path(P, 0, 1, mode=fw.FW_PATH_LAST_K)          # LAST_K needs D
    Pc = P.copy()
    Pc[3, 9] = 5
    Pc[5, 9] = 3                                             # a 3 <-> 5 cycle on the way to 9
    with pytest.raises(fw.FwError) as e:
        fw.fw_path(Pc, 3, 9)
    assert e.value.code == fw.FW_EINVAL
    # max_len smaller than the path: -FW_ERANGE, the first max_len vertices written
    lib = ctypes.CDLL(fw.library_path())
    lib.fw_path.restype = ctypes.c_int64
    lib.fw_path.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                            ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64]
    Wr = gen.ring(30, 1, dtype=np.int32)
    Dr, Pr = oracle.fw(Wr, "next")
    buf = (ctypes.c_int32 * 4)()
    r = lib.fw_path(Pr.ctypes.data, None, 0, 30, 0, 10, 0, ctypes.addressof(buf), 4)
    assert r == -fw.FW_ERANGE and list(buf) == [0, 1, 2, 3]

"""GPU parity: the CUDA path (through the C ABI, include/fw.h) against the CPU oracle
(oracle/) on seeded synthetic inputs. BASELINE.json north_star correctness requirements:
bit-exact D for integer-valued weights, rel 1e-5 for real FP32, P validated by
reconstructing paths (never bitwise: ties are legal), Dijkstra rows at n >= 16384.
"""
import numpy as np
import pytest

import apsp_inputs as gen
import oracle
from helpers import INF, assert_D_matches, exact_data, next_consistency

pytestmark = pytest.mark.gpu

fw = pytest.importorskip("paper_1811_01201_b200")
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


class Ctx:
    def __init__(self, flags):
        self.flags = flags

    def __enter__(self):
        fw.fw_init(0, self.flags)
        return self

    def __exit__(self, *a):
        fw.fw_free()


def solve(W, block=0, path="next", device=False):
    """Run the CUDA path on W (numpy); returns (D, P or None)."""
    flags = fw.FW_PATH_LAST_K if path == "lastk" else 0
    D = W.copy()
    P = np.empty(W.shape, dtype=np.int32) if path else None
    with Ctx(flags):
        if device:
            dD = torch.from_numpy(D).cuda()
            dP = torch.from_numpy(P).cuda() if P is not None else None
            f = fw.fw_solve_device_i32 if W.dtype == np.int32 else fw.fw_solve_device_f32
            f(dD, dP, block=block, stream=torch.cuda.current_stream())
            D = dD.cpu().numpy()
            P = dP.cpu().numpy() if dP is not None else None
        else:
            f = fw.fw_solve_i32 if W.dtype == np.int32 else fw.fw_solve
            f(D, P, block=block)
    return D, P


def check_against_oracle(W, block, path="next", device=False):
    D, P = solve(W, block, path, device)
    Dref, _ = oracle.fw(W, None)
    exact = exact_data(W)
    assert_D_matches(D, Dref, exact)
    if path:
        bad, first = oracle.check_paths(W, D, P, rtol=0.0 if exact else 1e-5, mode=path)
        assert bad == 0, f"{bad} invalid paths, first at {divmod(first, W.shape[0])}"
    return D, P


# ---- sizes spanning several tiles with ragged tails, every block size, both types ----
SIZES = [1, 2, 3, 31, 33, 127, 129, 200, 257, 383, 513]


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("block", [32, 64, 128])
def test_complete_int_f32(n, block):
    check_against_oracle(gen.generate("complete_int", n, 100 + n), block)


@pytest.mark.parametrize("n", [65, 300, 640])
@pytest.mark.parametrize("block", [32, 64, 128])
def test_complete_real_f32(n, block):
    check_against_oracle(gen.generate("complete_real", n, 200 + n), block)


@pytest.mark.parametrize("n,p", [(100, 0.02), (257, 0.01), (500, 0.004), (700, 0.1)])
@pytest.mark.parametrize("block", [32, 128])
def test_er_int32_unreachable(n, p, block):
    W = gen.generate("er_int", n, 300 + n, p=p, lo=1, hi=1000)
    D, _ = check_against_oracle(W, block)
    if p <= 0.01:
        assert (D == INF).any()           # INF outputs really exercised (reading C-14)


@pytest.mark.parametrize("n,p", [(333, 0.01), (450, 0.05)])
def test_er_f32_inf(n, p):
    D, P = check_against_oracle(gen.generate("er_int_f32", n, 400 + n, p=p, lo=1, hi=1000), 64)
    assert np.isinf(D).any() == (p < 0.03)
    assert ((P == -1) == (np.isinf(D))).all()


@pytest.mark.parametrize("n", [100, 385])
@pytest.mark.parametrize("block", [32, 128])
def test_lastk_mode(n, block):
    check_against_oracle(gen.generate("complete_int", n, 500 + n), block, path="lastk")
    check_against_oracle(gen.generate("er_int", n, 501 + n, p=0.02, lo=1, hi=1000), block, path="lastk")


@pytest.mark.parametrize("n", [64, 250, 512])
def test_distance_only(n):
    W = gen.generate("complete_real", n, 600 + n)
    D, P = solve(W, 64, path=None)
    assert P is None
    assert_D_matches(D, oracle.fw(W, None)[0], exact=False)


@pytest.mark.parametrize("n", [128, 256, 300])
@pytest.mark.parametrize("dtype", [np.float32, np.int32])
def test_device_entry(n, dtype):
    kind = "complete_int" if dtype == np.float32 else "er_int"
    W = gen.generate(kind, n, 700 + n, p=0.05, lo=1, hi=100)
    check_against_oracle(W, 0, device=True)


def test_device_entry_ld_and_stream():
    """d_dist with a leading dimension > n, on a side stream."""
    n, ld = 200, 256
    W = gen.generate("complete_int", n, 42)
    big = np.full((n, ld), 123.0, dtype=np.float32)
    big[:, :n] = W
    dD = torch.from_numpy(big).cuda()
    dP = torch.full((n, ld), -7, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with Ctx(0):
        fw.fw_solve_device_f32(dD, dP, n=n, ld=ld, block=64, stream=s)
    D = dD.cpu().numpy()
    P = dP.cpu().numpy()
    assert (D[:, n:] == 123.0).all() and (P[:, n:] == -7).all()     # padding columns untouched
    Dref, _ = oracle.fw(W, None)
    np.testing.assert_array_equal(D[:, :n], Dref)
    assert oracle.check_paths(W, D[:, :n].copy(), P[:, :n].copy())[0] == 0


# ---- closed forms and degenerate cases ------------------------------------------------
@pytest.mark.parametrize("n", [1, 2, 130, 1000])
def test_ring(n):
    W = gen.ring(n, 1)
    D, P = solve(W, 64)
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    np.testing.assert_array_equal(D, ((j - i) % n).astype(np.float32))
    np.testing.assert_array_equal(P, np.where(i == j, i, (i + 1) % n))


def test_abs_diff_and_uniform():
    n = 300
    W = gen.abs_diff(n)
    D, P = solve(W, 32)
    np.testing.assert_array_equal(D, W)
    np.testing.assert_array_equal(P, np.broadcast_to(np.arange(n), (n, n)))
    U = gen.uniform_complete(257, 5.0)
    D, P = solve(U, 128)
    np.testing.assert_array_equal(D, U)


def test_empty_graph_and_two_components():
    E = gen.empty_graph(150, np.int32)
    D, P = solve(E, 32)
    np.testing.assert_array_equal(D, E)
    assert (P[~np.eye(150, dtype=bool)] == -1).all() and (np.diag(P) == np.arange(150)).all()
    W = gen.two_components(400, 9, p=0.05)
    D, _ = check_against_oracle(W, 64)
    assert (D[:200, 200:] == INF).all() and (D[200:, :200] == INF).all()


def test_diagonal_forced_zero():
    W = gen.generate("complete_int", 70, 3)
    np.fill_diagonal(W, 55.0)
    D, P = solve(W, 32)
    assert (np.diag(D) == 0).all()
    W0 = W.copy()
    np.fill_diagonal(W0, 0)
    np.testing.assert_array_equal(D, oracle.fw(W0, None)[0])


def test_block_size_invariance_integer():
    """Integer data: D bitwise identical across BS (reading C-6)."""
    W = gen.generate("er_int", 450, 77, p=0.03, lo=1, hi=1000)
    Ds = [solve(W, b)[0] for b in (32, 64, 128)]
    assert all(np.array_equal(Ds[0], d) for d in Ds[1:])


def test_determinism(monkeypatch):
    """The stream-ordered schedule is deterministic bit for bit. The persistent launch (the default
    for small round-tag solves) takes its items dynamically and may read an operand tile after its
    owner has already relaxed it for a later round (reading R16): integer data stay
    bitwise (every sum is exact), real data agree run to run within the tolerance (rel 1e-5) with
    valid paths."""
    W = gen.generate("complete_real", 513, 5)
    monkeypatch.setenv("FW_PERSISTENT", "0")
    a = solve(W, 128)
    b = solve(W, 128)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])
    monkeypatch.setenv("FW_PERSISTENT", "1")
    c = solve(W, 128)
    d = solve(W, 128)
    np.testing.assert_allclose(c[0], a[0], rtol=1e-5)
    np.testing.assert_allclose(d[0], c[0], rtol=1e-5)
    for D, P in (c, d):
        assert oracle.check_paths(W, D, P, rtol=1e-5)[0] == 0
    Wi = gen.generate("complete_int", 513, 5)
    e, f = solve(Wi, 128), solve(Wi, 128)
    np.testing.assert_array_equal(e[0], f[0])


# ---- validation / error contract (fw.h) -----------------------------------------------
def test_validation_errors_leave_outputs_untouched():
    n = 40
    with Ctx(0):
        for bad in (-1.0, np.nan):
            W = gen.generate("complete_int", n, 1)
            W[3, 5] = bad
            D = W.copy()
            P = np.full((n, n), 77, dtype=np.int32)
            with pytest.raises(fw.FwError) as e:
                fw.fw_solve(D, P, block=32)
            assert e.value.code == fw.FW_EINVAL
            np.testing.assert_array_equal(np.isnan(D), np.isnan(W))
            np.testing.assert_array_equal(D[~np.isnan(W)], W[~np.isnan(W)])
            assert (P == 77).all()
        Wi = gen.generate("er_int", n, 2, p=0.5, lo=1, hi=10)
        Wi[1, 2] = INF + 1
        with pytest.raises(fw.FwError) as e:
            fw.fw_solve_i32(Wi.copy(), None, block=32)
        assert e.value.code == fw.FW_EINVAL
        Wi[1, 2] = 40_000_000            # (n-1) * w >= INF -> FW_ERANGE
        with pytest.raises(fw.FwError) as e:
            fw.fw_solve_i32(Wi.copy(), None, block=32)
        assert e.value.code == fw.FW_ERANGE
        with pytest.raises(fw.FwError) as e:
            fw.fw_solve(gen.generate("complete_int", n, 1), None, block=48)
        assert e.value.code == fw.FW_EINVAL
        with pytest.raises(fw.FwError) as e:
            fw.fw_solve(np.zeros((4, 4), np.float32), None, block=0, ngpus=2)
        assert e.value.code == fw.FW_EINVAL
    with pytest.raises(fw.FwError):
        fw.fw_solve(np.zeros((4, 4), np.float32))   # after fw_free: FW_ESTATE


def test_stats_and_timing():
    W = gen.generate("complete_int", 1000, 8)
    with Ctx(fw.FW_TIMING):
        D = W.copy()
        P = np.empty_like(W, dtype=np.int32)
        fw.fw_solve(D, P, block=128)
        s = fw.fw_last_stats()
    assert s.n == 1000 and s.n_pad == 1024 and s.block == 128 and s.rounds == 8
    assert s.solve_ms > 0 and s.phase3_ms > 0 and s.phase1_ms > 0 and s.post_ms >= 0
    assert s.phase3_ms <= s.solve_ms


# ---- BASELINE.json configs ---------------------------------------------------------------
def test_config_C1_full():
    """configs[0]: n=512 complete, FP32 integers [1,100], tile 32: bit-exact D, all paths."""
    W = gen.config_matrix("C1")
    check_against_oracle(W, 32)


def test_config_C2_full_oracle():
    """configs[1]: n=4096 complete, real [1,100), BS=128: rel 1e-5, paths for all pairs."""
    W = gen.config_matrix("C2")
    check_against_oracle(W, 128)


def _dijkstra_rows_check(W, D, P, seed, exact, count=64):
    src = gen.sources(W.shape[0], seed, count)
    R = oracle.dijkstra(W, src)
    Dr = D[src]
    if W.dtype == np.int32:
        np.testing.assert_array_equal(Dr.astype(np.int64), R)
    elif exact:
        np.testing.assert_array_equal(Dr.astype(np.float64), R)
    else:
        rel = np.abs(Dr.astype(np.float64) - R) / np.maximum(1.0, np.abs(R))
        assert np.array_equal(np.isinf(Dr), np.isinf(R)) and rel[np.isfinite(R)].max() <= 1e-5
    bad, first = oracle.check_paths(W, D, P, rows=src, rtol=0.0 if exact else 1e-5)
    assert bad == 0, f"{bad} bad paths from the seeded sources, first {first}"


def test_config_C3_er_int32():
    """configs[2]: n=8192 ER p=0.1 INT32 [1,1000]. n < 16384, so no sampling (BJ north_star):
    D bit-exact against the FULL oracle triple loop on every entry, every next-hop path of
    all n^2 pairs reconstructed and summed to D, plus 64 Dijkstra rows (independent)."""
    c = gen.CONFIGS["C3"]
    W = gen.config_matrix("C3")
    D, P = solve(W, 128)
    Dref, _ = oracle.fw(W, None)
    assert_D_matches(D, Dref, exact=True)
    bad, first = oracle.check_paths(W, D, P)
    assert bad == 0, f"{bad} invalid next-hop paths, first at {divmod(first, W.shape[0])}"
    _dijkstra_rows_check(W, D, P, c["seed"], True)


def test_config_C3_device_lastk_full():
    """C3 through the device entry in LAST_K mode: full-oracle D bitwise, all LAST_K paths."""
    W = gen.config_matrix("C3")
    D, P = solve(W, 128, path="lastk", device=True)
    Dref, _ = oracle.fw(W, None)
    assert_D_matches(D, Dref, exact=True)
    bad, first = oracle.check_paths(W, D, P, mode="lastk")
    assert bad == 0, f"{bad} invalid LAST_K paths, first at {divmod(first, W.shape[0])}"


def test_config_C3_sparse_unreachable():
    """Supplementary C3' (reading C-14): sparse ER so INF outputs and next = -1 occur."""
    W = gen.generate("er_int", 4096, 33, p=0.0004, lo=1, hi=1000)
    D, P = solve(W, 128)
    assert (D == INF).any()
    _dijkstra_rows_check(W, D, P, 33, True)
    assert next_consistency(W, D, P, exact=True) == 0


@pytest.mark.slow
def test_config_C4_16384():
    """configs[3]: n=16384 complete, FP32 integers: Dijkstra rows bitwise, next O(n^2)."""
    c = gen.CONFIGS["C4"]
    W = gen.config_matrix("C4")
    D, P = solve(W, 128)
    _dijkstra_rows_check(W, D, P, c["seed"], True)
    assert next_consistency(W, D, P, exact=True) == 0


@pytest.mark.slow
def test_config_C4_full_oracle():
    """configs[3] against the FULL oracle triple loop (n^3 = 4.4e12 relaxations on the host
    cores, a few minutes): D bitwise on all 2.7e8 entries, every next-hop path of every pair
    reconstructed and summed to D. Beyond north_star's 64-source requirement at n >= 16384."""
    W = gen.config_matrix("C4")
    D, P = solve(W, 128)
    Dref, _ = oracle.fw(W, None)
    assert_D_matches(D, Dref, exact=True)
    del Dref
    bad, first = oracle.check_paths(W, D, P)
    assert bad == 0, f"{bad} invalid next-hop paths, first at {divmod(first, W.shape[0])}"


@pytest.mark.slow
def test_config_C5_32768():
    """configs[4]: n=32768 complete, real FP32 [1,100) (4 GiB D + 4 GiB P) on one GPU —
    the 1-GPU denominator of the multi-GPU speedup. Dijkstra from the 64 seeded sources
    within rel 1e-5 (exact double sums), the paths from those sources reconstructed through
    next within rel 1e-5, and the O(n) next-hop check on 256 sampled rows."""
    c = gen.CONFIGS["C5"]
    W = gen.config_matrix("C5")
    D, P = solve(W, 128)
    _dijkstra_rows_check(W, D, P, c["seed"], False)
    rows = np.sort(gen.sources(W.shape[0], c["seed"] + 100, 256))
    assert next_consistency(W, D, P, exact=False, rows=rows, chunk=64) == 0


@pytest.mark.slow
def test_paper_largest_n65536():
    """the paper's largest workload N=65536 (16 GiB D + 16 GiB P) with the
    configs[3] recipe (complete, FP32 integers [1,100]) on one GPU, device entry point:
    Dijkstra from 8 seeded sources bitwise, next-hop check on 64 sampled rows."""
    n, seed = 65536, 4
    dW = gen.generate_torch("complete_int", n, seed, device="cuda")
    W = dW.cpu().numpy()
    dP = torch.empty((n, n), dtype=torch.int32, device="cuda")
    with Ctx(fw.FW_TIMING):
        fw.fw_solve_device_f32(dW, dP, block=128, stream=torch.cuda.current_stream())
        s = fw.fw_last_stats()
    assert s.n_pad == n and s.rounds == n // 128 and s.p_method == 2
    D = dW.cpu().numpy()
    del dW
    P = dP.cpu().numpy()
    del dP
    src = gen.sources(n, seed, 8)
    np.testing.assert_array_equal(D[src].astype(np.float64), oracle.dijkstra(W, src))
    rows = np.sort(gen.sources(n, seed + 100, 64))
    assert next_consistency(W, D, P, exact=True, rows=rows, chunk=16) == 0


# ---- P method selection (reading R9): exact keyed arg-min vs round tags ---------------
def _solve_stats(W, block, flags=0):
    D = W.copy()
    P = np.empty(W.shape, dtype=np.int32)
    with Ctx(flags | fw.FW_TIMING):
        (fw.fw_solve_i32 if W.dtype == np.int32 else fw.fw_solve)(D, P, block=block)
        s = fw.fw_last_stats()
    return D, P, s


def test_keyed_mode_static_bound():
    """Complete integer graph: keys are provably exact (no INF entries)."""
    W = gen.generate("complete_int", 300, 11)
    D, P, s = _solve_stats(W, 64)
    assert s.p_method == 2
    np.testing.assert_array_equal(D, oracle.fw(W, None)[0])
    assert oracle.check_paths(W, D, P)[0] == 0


def test_keyed_mode_speculative_success():
    """ER graph with INF entries and (n-1)*max_w beyond the key range: the keyed run is
    speculative and verified by the max stored key (distances stay small)."""
    W = gen.generate("er_int_f32", 700, 12, p=0.1, lo=1, hi=1000)
    D, P, s = _solve_stats(W, 128)
    assert s.p_method == 2
    np.testing.assert_array_equal(D, oracle.fw(W, None)[0])
    assert oracle.check_paths(W, D, P)[0] == 0


@pytest.mark.parametrize("dtype", [np.float32, np.int32])
def test_keyed_mode_fallback_to_tags(dtype):
    """Ring with weight 1000 (FP32) / 40000 (INT32): distances leave the exact key range,
    the solve is redone with round tags and must still be exact."""
    n = 1000 if dtype == np.float32 else 200
    w = 1000 if dtype == np.float32 else 40000
    W = gen.ring(n, w, dtype)
    D, P, s = _solve_stats(W, 64)
    assert s.p_method == 1
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    np.testing.assert_array_equal(D.astype(np.int64), ((j - i) % n) * w)
    np.testing.assert_array_equal(P, np.where(i == j, i, (i + 1) % n))


def test_real_weights_use_tags():
    W = gen.generate("complete_real", 256, 13)
    D, P, s = _solve_stats(W, 64)
    assert s.p_method == 1
    assert_D_matches(D, oracle.fw(W, None)[0], exact=False)
    assert oracle.check_paths(W, D, P, rtol=1e-5)[0] == 0


def test_keyed_lastk():
    W = gen.generate("er_int", 513, 14, p=0.05, lo=1, hi=1000)
    D, P, s = _solve_stats(W, 32, fw.FW_PATH_LAST_K)
    assert s.p_method == 2
    np.testing.assert_array_equal(D, oracle.fw(W, None)[0])
    assert oracle.check_paths(W, D, P, mode="lastk")[0] == 0


@pytest.mark.parametrize("n,hi,p,block,want_f32", [
    (700, 1000, 0.1, 128, 1),       # C3-like: keys fit FP32 (speculative, verified)
    (300, 3000, 0.05, 64, 1),       # larger weights, keys still below 2^24 after the solve
    (257, 3_000_000, 0.05, 32, 0),  # (n-1)*max_w >= 2^24 and keys out of FP32 range: INT32 compute
])
def test_int32_compute_type(n, hi, p, block, want_f32):
    """INT32 data relaxes in FP32 when every stored value is an integer below 2^24 (DESIGN.md
    §4.7), natively otherwise; D bit-exact and paths valid either way."""
    W = gen.generate("er_int", n, 21, p=p, lo=1, hi=hi)
    for path in ("next", None):
        D = W.copy()
        P = np.empty(W.shape, dtype=np.int32) if path else None
        with Ctx(fw.FW_TIMING):
            fw.fw_solve_i32(D, P, block=block)
            s = fw.fw_last_stats()
        if path or want_f32 == 0:
            assert s.compute_f32 == want_f32, (s.compute_f32, s.p_method)
        np.testing.assert_array_equal(D, oracle.fw(W, None)[0])
        if path:
            assert oracle.check_paths(W, D, P)[0] == 0


def test_zero_weight_edges_distances():
    """Zero off-diagonal weights are in the domain (reading C-5): D must be exact."""
    W = gen.generate("er_int_f32", 260, 15, p=0.05, lo=0, hi=3)
    D, P = solve(W, 64)
    np.testing.assert_array_equal(D, oracle.fw(W, None)[0])


# ---- one context, many solves: workspace growth/shrink, per-kernel configuration, counters -
def test_mixed_sequence_one_context():
    """A seeded sequence of solves through ONE fw_init context: sizes up and down, every block
    size, FP32 integer / real / INF data and INT32, next-hop / LAST_K / distance-only, host and
    device entry points — each checked against the oracle (catches state carried between solves:
    workspaces, lazily configured kernel attributes, look-ahead counters, key fallbacks)."""
    rng = np.random.default_rng(2024)
    kinds = ["complete_int", "complete_real", "er_int", "er_int_f32", "er_real"]
    with Ctx(fw.FW_TIMING):
        for step in range(24):
            n = int(rng.choice([1, 5, 64, 129, 300, 520, 1100]))
            kind = kinds[step % len(kinds)]
            block = int(rng.choice([0, 32, 64, 128]))
            W = gen.generate(kind, n, 900 + step, p=0.05, lo=1, hi=int(rng.choice([9, 1000])))
            path = [None, "next"][step % 2]
            device = bool(step % 3 == 0)
            D = W.copy()
            P = np.empty(W.shape, dtype=np.int32) if path else None
            if device:
                dD = torch.from_numpy(D).cuda()
                dP = torch.from_numpy(P).cuda() if P is not None else None
                f = fw.fw_solve_device_i32 if W.dtype == np.int32 else fw.fw_solve_device_f32
                f(dD, dP, block=block, stream=torch.cuda.current_stream())
                D = dD.cpu().numpy()
                P = dP.cpu().numpy() if dP is not None else None
            else:
                (fw.fw_solve_i32 if W.dtype == np.int32 else fw.fw_solve)(D, P, block=block)
            exact = exact_data(W)
            assert_D_matches(D, oracle.fw(W, None)[0], exact)
            if path:
                bad, first = oracle.check_paths(W, D, P, rtol=0.0 if exact else 1e-5)
                assert bad == 0, (step, kind, n, block, bad, first)


@pytest.mark.parametrize("kind,path", [("complete_int", "next"), ("complete_real", "lastk"),
                                       ("er_int", "next"), ("er_int", "lastk")])
def test_fw_path_on_gpu_results(kind, path):
    """fw_path (host-only) reconstructs shortest paths from the P the GPU solve returned: every
    sampled path starts at i, ends at j, uses edges of W, and its weights sum to D[i][j]
    (exactly for integer data, rel 1e-5 for reals); unreachable pairs give []."""
    n = 300
    W = gen.generate(kind, n, 777, p=0.02, lo=1, hi=50)
    D, P = solve(W, 128, path)
    mode = fw.FW_PATH_LAST_K if path == "lastk" else fw.FW_PATH_NEXT_HOP
    rng = np.random.default_rng(7)
    w = W.astype(np.float64)
    if W.dtype == np.int32:
        w[W >= INF] = np.inf
    Dd = D.astype(np.float64)
    if W.dtype == np.int32:
        Dd[D >= INF] = np.inf
    for i, j in rng.integers(0, n, size=(400, 2)):
        p = fw.fw_path(P, int(i), int(j), mode, dist=D)
        if not np.isfinite(Dd[i, j]):
            assert p == []
            continue
        assert p[0] == i and p[-1] == j and len(set(p)) == len(p)
        s = sum(w[a, b] for a, b in zip(p, p[1:]))
        assert abs(s - Dd[i, j]) <= 1e-5 * max(1.0, Dd[i, j]), (i, j, s, Dd[i, j])


# ---- two rounds per phase-3 pass: keyed / plain solves, BS = 128, R even ----
@pytest.mark.parametrize("kind,n,path", [("complete_int", 512, "next"), ("complete_int", 700, "next"),
                                         ("complete_int", 1000, "lastk"), ("complete_real", 768, None),
                                         ("er_int", 1024, "next"), ("er_int_f32", 900, "next")])
def test_pair_rounds_against_oracle(kind, n, path, monkeypatch):
    """Pairs of rounds (strip region by two sub-rounds, bulk through 256 k in one pass): D
    bit-exact against the oracle (rel 1e-5 for reals) and paths valid; D identical to the
    one-round-per-pass schedule (FW_PAIRS=0) for integer data."""
    W = gen.generate(kind, n, 990 + n, p=0.02, lo=1, hi=1000)
    D, P = solve(W, 128, path)
    exact = exact_data(W)
    assert_D_matches(D, oracle.fw(W, None)[0], exact)
    if path:
        bad, first = oracle.check_paths(W, D, P, rtol=0.0 if exact else 1e-5, mode=path)
        assert bad == 0, f"{bad} invalid paths, first at {divmod(first, n)}"
    monkeypatch.setenv("FW_PAIRS", "0")
    D0, _ = solve(W, 128, path)
    if exact:
        np.testing.assert_array_equal(D, D0)


def test_pair_rounds_ring_closed_form():
    """Ring + chords (long chains through every block) under the pair schedule."""
    n = 1280
    W = gen.ring_with_chords(n, 5, 300)
    D, P = solve(W, 128, "next")
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    np.testing.assert_array_equal(D, ((j - i) % n).astype(np.float32))
    np.testing.assert_array_equal(P, np.where(i == j, i, (i + 1) % n))


@pytest.mark.parametrize("n", [768, 1000])
def test_pair_rounds_int32_native_keys(n):
    """INT32 weights above the FP32 key range (max_w > 32766), no INF: native INT32 keys
    (VIADDMNMX) under two rounds per pass; bit-exact against the oracle, paths valid."""
    W = gen.generate("er_int", n, 995 + n, p=1.0, lo=1, hi=200000)
    D, P, s = _solve_stats(W, 128)
    assert s.p_method == 2 and s.compute_f32 == 0 and s.phase3_launches < s.rounds
    np.testing.assert_array_equal(D, oracle.fw(W, None)[0])
    assert oracle.check_paths(W, D, P)[0] == 0


# ---- programmatic dependent launch of consecutive phase-3 launches ----------
@pytest.mark.parametrize("kind,n,path,pairs", [("complete_int", 1024, "next", "1"),
                                               ("complete_int", 1000, "lastk", "0"),
                                               ("complete_real", 1280, "next", "1"),
                                               ("complete_real", 900, "next", "0"),
                                               ("er_int", 1152, "next", "1")])
@pytest.mark.parametrize("device", [True, False])
def test_pdl_schedule_identical(kind, n, path, pairs, device, monkeypatch):
    """Phase-3 launches overlapping the previous launch's last wave (main loop before
    griddepcontrol.wait) give bitwise the same D and P as stream-ordered launches (FW_PDL=0):
    every tile sees the same operands and the same order of rounds. Checked against the
    oracle too; device entry point (one solve) and host entry point (row-chunk pipeline).
    The stream-ordered schedule is pinned (FW_PERSISTENT=0): PDL does not apply to the persistent
    launch, whose dynamic item order gives real-valued data ulp-level differences between runs
    ("Overlapping rounds")."""
    monkeypatch.setenv("FW_PAIRS", pairs)
    monkeypatch.setenv("FW_PERSISTENT", "0")
    W = gen.generate(kind, n, 1200 + n, p=0.05, lo=1, hi=1000)
    D1, P1 = solve(W, 128, path, device=device)
    monkeypatch.setenv("FW_PDL", "0")
    D0, P0 = solve(W, 128, path, device=device)
    np.testing.assert_array_equal(D1, D0)
    np.testing.assert_array_equal(P1, P0)
    exact = exact_data(W)
    assert_D_matches(D1, oracle.fw(W, None)[0], exact)
    bad, first = oracle.check_paths(W, D1, P1, rtol=0.0 if exact else 1e-5, mode=path)
    assert bad == 0, f"{bad} invalid paths, first at {divmod(first, n)}"


@pytest.mark.parametrize("opt", ["lookahead", "pairs", "pdl", "pair_order"])
def test_set_option_schedules_identical_D(opt):
    """fw_set_option switches the schedule of the live context: the distances stay identical
    (integer data) and P stays a valid next hop."""
    W = gen.generate("complete_int", 1024, 55)
    out = []
    for v in (1, 0):
        D = W.copy()
        P = np.empty(W.shape, dtype=np.int32)
        with Ctx(0):
            fw.fw_set_option(opt, v)
            fw.fw_solve(D, P, block=128)
        out.append(D)
        assert oracle.check_paths(W, D, P)[0] == 0
    np.testing.assert_array_equal(out[0], out[1])
    with Ctx(0):
        with pytest.raises(fw.FwError):
            fw.fw_set_option("no_such_option", 1)


# ---- one persistent launch per solve (fw_persist.cuh) ----------
PERSIST_CASES = [
    ("complete_int", 129, "next"), ("complete_int", 640, "next"), ("complete_int", 1000, "lastk"),
    ("complete_real", 300, "next"), ("complete_real", 777, "next"), ("complete_real", 1024, "lastk"),
    ("er_int", 700, "next"), ("er_int", 513, "lastk"), ("er_int_f32", 900, "next"),
    ("complete_int", 600, None), ("complete_real", 500, None),
]


@pytest.mark.parametrize("kind,n,path", PERSIST_CASES)
@pytest.mark.parametrize("device", [False, True])
def test_persistent_against_oracle(kind, n, path, device):
    """The whole solve as one persistent launch (work items in round order, per-tile round
    counters) for every P method (FP32 keys, INT32 keys / tags, round tags, distance only):
    D against the oracle (bitwise for integer data), P valid by reconstruction; for integer
    data D bitwise equal to the stream-ordered schedule."""
    W = gen.generate(kind, n, 900 + n, p=0.02, lo=1, hi=1000 if kind.startswith("er") else 100)
    flags = (fw.FW_PATH_LAST_K if path == "lastk" else 0) | fw.FW_TIMING
    out = {}
    for persist in (1, 0):
        D = W.copy()
        P = np.empty(W.shape, dtype=np.int32) if path else None
        with Ctx(flags):
            fw.fw_set_option("persistent", persist)
            if device:
                dD = torch.from_numpy(D).cuda()
                dP = torch.from_numpy(P).cuda() if P is not None else None
                f = fw.fw_solve_device_i32 if W.dtype == np.int32 else fw.fw_solve_device_f32
                f(dD, dP, block=128, stream=torch.cuda.current_stream())
                D = dD.cpu().numpy()
                P = dP.cpu().numpy() if dP is not None else None
            else:
                fw.fw_set_host_pipeline(0)
                (fw.fw_solve_i32 if W.dtype == np.int32 else fw.fw_solve)(D, P, block=128)
            s = fw.fw_last_stats()
        assert s.persistent == persist
        out[persist] = (D, P)
    D, P = out[1]
    exact = exact_data(W)
    assert_D_matches(D, oracle.fw(W, None)[0], exact)
    if path:
        bad, first = oracle.check_paths(W, D, P, rtol=0.0 if exact else 1e-5, mode=path)
        assert bad == 0, f"{bad} invalid paths, first at {divmod(first, n)}"
    if exact:
        np.testing.assert_array_equal(D, out[0][0])


@pytest.mark.parametrize("gap", [0, 1, 7, 100000])
def test_persistent_gap_extremes(gap):
    """Any position of the next round's phase-2 items in the work order is correct (the order only
    decides how long items wait): P2(K+1) right after P1(K+1), or after all of round K."""
    W = gen.generate("complete_real", 896, 5)
    D = W.copy()
    P = np.empty(W.shape, dtype=np.int32)
    with Ctx(0):
        fw.fw_set_option("persistent", 1)
        fw.fw_set_option("persist_gap", gap)
        fw.fw_set_host_pipeline(0)
        fw.fw_solve(D, P, block=128)
    assert_D_matches(D, oracle.fw(W, None)[0], False)
    assert oracle.check_paths(W, D, P, rtol=1e-5)[0] == 0


def test_persistent_ring_closed_form():
    """Long chains (every path through many rounds): ring of weight 1, n = 1000."""
    n = 1000
    W = gen.ring(n, 1)
    D = W.copy()
    P = np.empty(W.shape, dtype=np.int32)
    with Ctx(0):
        fw.fw_set_option("persistent", 1)
        fw.fw_set_host_pipeline(0)
        fw.fw_solve(D, P, block=128)
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    np.testing.assert_array_equal(D.astype(np.int64), (j - i) % n)
    np.testing.assert_array_equal(P, np.where(i == j, i, (i + 1) % n))


# ---- asynchronous device solve (fw_set_option("async", 1)): no validation, no host round trip ----
@pytest.mark.parametrize("kind,n", [("complete_int", 640), ("complete_real", 513), ("er_int", 700),
                                    ("complete_int", 3000), ("complete_real", 4096)])
def test_async_device_solve(kind, n):
    """The asynchronous device entry returns once the solve is enqueued; after the stream is
    synchronised D matches the oracle (bitwise for integer data) and P is valid; fw_last_stats
    waits for the solve and reports its time."""
    W = gen.generate(kind, n, 400 + n, p=0.02, lo=1, hi=1000 if kind.startswith("er") else 100)
    with Ctx(0):
        fw.fw_set_option("async", 1)
        dD = torch.from_numpy(W).cuda()
        dP = torch.empty(W.shape, dtype=torch.int32, device="cuda")
        f = fw.fw_solve_device_i32 if W.dtype == np.int32 else fw.fw_solve_device_f32
        s = torch.cuda.Stream()
        f(dD, dP, block=0, stream=s)
        s.synchronize()
        st = fw.fw_last_stats()
        D, P = dD.cpu().numpy(), dP.cpu().numpy()
    assert st.solve_ms > 0 and st.p_method == 1
    exact = exact_data(W)
    assert_D_matches(D, oracle.fw(W, None)[0], exact)
    bad, first = oracle.check_paths(W, D, P, rtol=0.0 if exact else 1e-5)
    assert bad == 0, f"{bad} invalid paths, first at {divmod(first, n)}"


@pytest.mark.parametrize("kind,n", [("complete_int", 1024), ("complete_real", 2048)])
def test_async_solve_captured_in_cuda_graph(kind, n):
    """With the workspaces allocated by a warm-up solve, an asynchronous solve captures into a
    CUDA graph; replaying the graph on a fresh copy of the input gives the oracle's D."""
    W = gen.generate(kind, n, 77 + n)
    dW = torch.from_numpy(W).cuda()
    dD = dW.clone()
    dP = torch.empty(W.shape, dtype=torch.int32, device="cuda")
    with Ctx(0):
        fw.fw_set_option("async", 1)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            fw.fw_solve_device_f32(dD, dP, block=128, stream=s)   # warm-up: allocations, attributes
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
            dD.copy_(dW)
            fw.fw_solve_device_f32(dD, dP, block=128, stream=s)
        dD.fill_(0)
        g.replay()
        torch.cuda.synchronize()
        D, P = dD.cpu().numpy(), dP.cpu().numpy()
    exact = exact_data(W)
    assert_D_matches(D, oracle.fw(W, None)[0], exact)
    assert oracle.check_paths(W, D, P, rtol=0.0 if exact else 1e-5)[0] == 0


@pytest.mark.parametrize("path", ["next", "lastk"])
def test_persistent_int32_keys(path):
    """Weights up to 100000 rule out FP32 keys (key range 32766) but not INT32 keys (2097150):
    the persistent launch runs the INT32 keyed items (phase 1 with the per-step P select)."""
    n = 600
    W = gen.generate("er_int", n, 91, p=1.0, lo=1, hi=100000)
    D = W.copy()
    P = np.empty(W.shape, dtype=np.int32)
    with Ctx(fw.FW_PATH_LAST_K if path == "lastk" else 0):
        fw.fw_set_option("persistent", 1)
        fw.fw_set_host_pipeline(0)
        fw.fw_solve_i32(D, P, block=128)
        s = fw.fw_last_stats()
    assert s.persistent == 1 and s.p_method == 2 and s.compute_f32 == 0
    np.testing.assert_array_equal(D, oracle.fw(W, None)[0])
    assert oracle.check_paths(W, D, P, mode=path)[0] == 0


@pytest.mark.parametrize("lone", [0, 1])
@pytest.mark.parametrize("kind,n", [("complete_real", 2000), ("complete_int", 1536), ("er_int", 1100)])
def test_persistent_dedicated_phase1_cta(kind, n, lone):
    """The one-GPU persistent launch with and without the dedicated phase-1 CTA (one SM keeps a
    single CTA that runs every P1 item; the others skip them): D against the oracle, paths valid."""
    W = gen.generate(kind, n, 40 + n, p=0.05, lo=1, hi=1000 if kind.startswith("er") else 100)
    fw.fw_init(0, 0)
    try:
        fw.fw_set_option("persistent", 1)
        fw.fw_set_option("persist_p1_lone", lone)
        dD = torch.from_numpy(W).cuda()
        dP = torch.empty(W.shape, dtype=torch.int32, device="cuda")
        (fw.fw_solve_device_i32 if W.dtype == np.int32 else fw.fw_solve_device_f32)(
            dD, dP, block=128, stream=torch.cuda.current_stream())
        s = fw.fw_last_stats()
    finally:
        fw.fw_free()
    assert s.persistent == 1
    D, P = dD.cpu().numpy(), dP.cpu().numpy()
    exact = exact_data(W)
    assert_D_matches(D, oracle.fw(W, None)[0], exact)
    bad, first = oracle.check_paths(W, D, P, rtol=0.0 if exact else 1e-5)
    assert bad == 0, (bad, divmod(first, n))

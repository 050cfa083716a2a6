"""GPU parity of the host pipeline (reading R16): fw_solve / fw_solve_i32 with
pinned host buffers split the rows into chunks whose H2D, rounds and D2H overlap. Against the
CPU oracle: D bit-exact for integer data (rel 1e-5 for reals), P valid by path reconstruction;
the speculative plan (taken from the first chunk) falls back to the standard solve when the
whole matrix needs another plan, and validation errors still leave the outputs untouched.
Small chunk sizes (fw_set_host_pipeline) make several chunks and ragged tails at oracle sizes.
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


def pinned(a: np.ndarray):
    t = torch.from_numpy(a.copy()).pin_memory()
    return t


def solve_pinned(W, chunk_tiles, path="next", block=128, pin=True):
    """fw_solve on pinned host tensors (pin=False: pageable NumPy arrays, staged through the
    library's pinned ring) with the given pipeline chunk; (D, P, stats)."""
    flags = fw.FW_PATH_LAST_K if path == "lastk" else 0
    if pin:
        hD = pinned(W)
        hP = torch.full(W.shape, -5, dtype=torch.int32).pin_memory() if path else None
    else:
        hD = torch.from_numpy(W.copy())
        hP = torch.full(W.shape, -5, dtype=torch.int32) if path else None
    fw.fw_init(0, flags)
    try:
        fw.fw_set_host_pipeline(chunk_tiles)
        f = fw.fw_solve_i32 if W.dtype == np.int32 else fw.fw_solve
        f(hD, hP, block=block)
        st = fw.fw_last_stats()
    finally:
        fw.fw_free()
    return hD.numpy(), (hP.numpy() if hP is not None else None), st


def check(W, chunk_tiles, path="next", expect_chunks=None, pin=True):
    D, P, st = solve_pinned(W, chunk_tiles, path, pin=pin)
    exact = exact_data(W)
    assert_D_matches(D, oracle.fw(W, None)[0], exact)
    if path:
        bad, first = oracle.check_paths(W, D, P, rtol=0.0 if exact else 1e-5, mode=path)
        assert bad == 0, f"{bad} invalid paths, first at {divmod(first, W.shape[0])}"
    if expect_chunks is not None:
        assert st.host_chunks == expect_chunks, st.host_chunks
    return D, P, st


@pytest.mark.parametrize("n,ct", [(256, 1), (300, 1), (513, 2), (777, 2), (1000, 3), (1024, 4)])
def test_pipeline_complete_int_f32(n, ct):
    tiles = (n + 127) // 128
    check(gen.generate("complete_int", n, 900 + n), ct, expect_chunks=-(-tiles // ct))


@pytest.mark.parametrize("n,ct", [(640, 1), (900, 2)])
def test_pipeline_int32_small_weights(n, ct):
    """INT32 data whose keys fit FP32 run through the FP32 keyed kernels in the pipeline."""
    W = gen.generate("er_int", n, 910 + n, p=1.0, lo=1, hi=100)
    D, P, st = check(W, ct, expect_chunks=-(-((n + 127) // 128) // ct))
    assert st.compute_f32 == 1


@pytest.mark.parametrize("n,ct", [(384, 1), (700, 2)])
def test_pipeline_lastk(n, ct):
    check(gen.generate("complete_int", n, 920 + n), ct, path="lastk",
          expect_chunks=-(-((n + 127) // 128) // ct))


@pytest.mark.parametrize("n,ct", [(500, 1), (1000, 2)])
def test_pipeline_distance_only_real(n, ct):
    """next = NULL: the PLAIN plan is always static, real weights pipeline too."""
    check(gen.generate("complete_real", n, 930 + n), ct, path=None,
          expect_chunks=-(-((n + 127) // 128) // ct))


def test_pipeline_closed_form_ring():
    """Ring + heavy chords at several chunks: D = (j - i) mod n, next = i + 1."""
    n = 1100
    W = np.full((n, n), np.float32(n), dtype=np.float32)
    i = np.arange(n)
    W[i, (i + 1) % n] = 1.0
    D, P, st = solve_pinned(W, 2)
    assert st.host_chunks == 5
    ii, jj = np.meshgrid(i, i, indexing="ij")
    np.testing.assert_array_equal(D, ((jj - ii) % n).astype(np.float32))
    np.testing.assert_array_equal(P, np.where(ii == jj, ii, (ii + 1) % n))


def test_pipeline_matches_standard_D():
    """Pipelined and unpipelined host solves give bitwise-identical D on integer data."""
    W = gen.generate("complete_int", 1280, 77)
    D1, P1, s1 = solve_pinned(W, 2)
    D0, P0, s0 = solve_pinned(W, 0)
    assert s1.host_chunks == 5 and s0.host_chunks == 0
    np.testing.assert_array_equal(D1, D0)
    assert next_consistency(W, D1, P1, exact=True) == 0


def test_pipeline_deterministic():
    W = gen.generate("complete_int", 900, 78)
    a = solve_pinned(W, 1)
    b = solve_pinned(W, 1)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])


def test_pipeline_fallback_real_weight_late():
    """Chunk 0 is integer-valued (keyed plan speculated) but a later chunk holds a real weight:
    the whole matrix needs round tags, so the pipelined work is dropped and the standard
    solve runs (host_chunks = 0); results still match the oracle."""
    n = 700
    W = gen.generate("complete_int", n, 940)
    W[600, 5] = np.float32(37.25)
    D, P, st = check(W, 1, expect_chunks=0)
    assert st.p_method == 1


def test_pipeline_fallback_inf_late():
    """A no-edge entry outside chunk 0 makes the key range speculative: standard path."""
    n = 640
    W = gen.generate("complete_int", n, 941)
    W[500, 3] = np.inf
    W[500, 4] = 1000.0     # (n-1) * max_w > 65534: the key range is no longer static
    check(W, 1, expect_chunks=0)


@pytest.mark.parametrize("n,ct,path", [(520, 1, "next"), (700, 2, "next"), (640, 1, "lastk")])
def test_pipeline_round_tags(n, ct, path):
    """Real weights with P (round tags): D leaves chunk by chunk, the tag post-pass runs on the
    whole final D after the last chunk (reading R9 holds for any round order), then P leaves."""
    D, P, st = check(gen.generate("complete_real", n, 942 + n), ct, path=path,
                     expect_chunks=-(-((n + 127) // 128) // ct))
    assert st.p_method == 1


def test_pipeline_round_tags_with_inf():
    """Real weights with no-edge entries (unreachable pairs) through the tag pipeline."""
    n = 600
    W = gen.generate("complete_real", n, 950)
    rng = np.random.default_rng(950)
    W[rng.random((n, n)) < 0.995] = np.inf
    np.fill_diagonal(W, 0)
    D, P, st = check(W, 1, expect_chunks=5)
    assert np.isinf(D).any()
    assert ((P == -1) == np.isinf(D)).all()


@pytest.mark.parametrize("bad", [-1.0, np.nan])
def test_pipeline_error_in_late_chunk_leaves_outputs(bad):
    """A negative / NaN weight in the last chunk: FW_EINVAL, dist and next untouched."""
    n = 600
    W = gen.generate("complete_int", n, 943)
    W[590, 17] = bad
    hD = pinned(W)
    hP = torch.full(W.shape, -5, dtype=torch.int32).pin_memory()
    fw.fw_init(0, 0)
    try:
        fw.fw_set_host_pipeline(1)
        with pytest.raises(fw.FwError) as e:
            fw.fw_solve(hD, hP, block=128)
        assert e.value.code == fw.FW_EINVAL
    finally:
        fw.fw_free()
    D = hD.numpy()
    np.testing.assert_array_equal(np.isnan(D), np.isnan(W))
    np.testing.assert_array_equal(D[~np.isnan(W)], W[~np.isnan(W)])
    assert (hP.numpy() == -5).all()


def test_pipeline_int32_erange_late():
    """INT32: a weight in a later chunk makes (n-1)*max_w reach INF: FW_ERANGE, untouched."""
    n = 520
    W = gen.generate("er_int", n, 944, p=1.0, lo=1, hi=100)
    W[515, 2] = 0x3FFFFFFF // 400
    hD = pinned(W)
    fw.fw_init(0, 0)
    try:
        fw.fw_set_host_pipeline(1)
        with pytest.raises(fw.FwError) as e:
            fw.fw_solve_i32(hD, None, block=128)
        assert e.value.code == fw.FW_ERANGE
    finally:
        fw.fw_free()
    np.testing.assert_array_equal(hD.numpy(), W)


@pytest.mark.parametrize("kind,n,ct,path", [("complete_int", 512, 1, "next"), ("complete_real", 700, 2, "next"),
                                             ("complete_int", 900, 2, "lastk"), ("complete_real", 640, 1, None),
                                             ("er_int", 1000, 1, "next")])
def test_pipeline_pageable(kind, n, ct, path):
    """Pageable (NumPy) host buffers: chunks are staged through the pinned ring by the copy
    pool, same parity as pinned buffers (keys, tags, LAST_K, D only, speculative INT32 keys)."""
    W = gen.generate(kind, n, 945 + n, p=0.05, lo=1, hi=1000) if kind == "er_int" else gen.generate(kind, n, 945 + n)
    check(W, ct, path=path, expect_chunks=-(-((n + 127) // 128) // ct), pin=False)


def test_pipeline_pageable_numpy_api():
    """The plain NumPy call a user makes: fw_solve(D, P) on pageable arrays, pipelined."""
    W = gen.generate("complete_int", 512, 946)
    D = W.copy()
    P = np.empty(W.shape, np.int32)
    fw.fw_init(0, 0)
    try:
        fw.fw_set_host_pipeline(1)
        fw.fw_solve(D, P, block=128)
        assert fw.fw_last_stats().host_chunks == 4
    finally:
        fw.fw_free()
    np.testing.assert_array_equal(D, oracle.fw(W, None)[0])
    bad, first = oracle.check_paths(W, D, P)
    assert bad == 0


@pytest.mark.slow
def test_pipeline_auto_c4_dijkstra_rows():
    """C4 (n = 16384, BASELINE configs[3]) through the auto pipeline (chunks of 8, 8, 16, 32, 64
    tile-rows):
    Dijkstra rows from 64 seeded sources bit-exact, next-hop consistency on those rows."""
    c = gen.CONFIGS["C4"]
    n = c["n"]
    W = gen.config_matrix("C4")
    hD = torch.from_numpy(W).pin_memory()
    hP = torch.empty((n, n), dtype=torch.int32).pin_memory()
    fw.fw_init(0, 0)
    try:
        fw.fw_solve(hD, hP, block=128)
        st = fw.fw_last_stats()
    finally:
        fw.fw_free()
    assert st.host_chunks == 5
    D, P = hD.numpy(), hP.numpy()
    src = gen.sources(n, c["seed"])
    np.testing.assert_array_equal(D[src].astype(np.float64), oracle.dijkstra(W, src))
    assert next_consistency(W, D, P, exact=True, rows=src) == 0


@pytest.mark.parametrize("n,p,ct", [(1000, 0.1, 1), (900, 0.003, 2)])
def test_pipeline_speculative_keys_er_int32(n, p, ct):
    """INT32 ER graphs with no-edge entries (BASELINE configs[2] recipe, small n): the key range
    is only speculatively exact ((n-1) * max_w > 65534), so each chunk is checked against the
    running max key before it leaves; here every check passes and the pipeline completes."""
    W = gen.generate("er_int", n, 960 + n, p=p, lo=1, hi=1000)
    D, P, st = check(W, ct, expect_chunks=-(-((n + 127) // 128) // ct))
    assert st.p_method == 2
    if p < 0.05:
        assert (D == INF).any()


def test_pipeline_speculative_keys_fail_falls_back():
    """A ring with weight 1000 stores distances up to 999000: FP32 keys leave the exact range,
    the first departure check fails before anything is copied out, and the standard solve runs
    from the device copy of the input (INT32 keys): D = ((j - i) mod n) * 1000, next = i + 1."""
    n = 1000
    W = gen.ring(n, 1000, dtype=np.int32)
    D, P, st = solve_pinned(W, 1)
    assert st.host_chunks == 0 and st.p_method == 2
    i = np.arange(n)
    ii, jj = np.meshgrid(i, i, indexing="ij")
    np.testing.assert_array_equal(D.astype(np.int64), ((jj - ii) % n) * 1000)
    np.testing.assert_array_equal(P, np.where(ii == jj, ii, (ii + 1) % n))


def test_pipeline_pageable_large_slices():
    """n = 5000 with chunks of 20 tile-rows (51 MB of D per chunk): every chunk copy is larger
    than one 32 MiB staging slice, so it is split over several slices of the ring."""
    n = 5000
    W = gen.generate("complete_int", n, 947)
    D, P, st = solve_pinned(W, 20, pin=False)
    assert st.host_chunks == 2
    src = gen.sources(n, 947, 16)
    np.testing.assert_array_equal(D[src].astype(np.float64), oracle.dijkstra(W, src))
    assert next_consistency(W, D, P, exact=True, rows=src) == 0


def test_pipeline_int32_native_keys():
    """INT32 weights above the FP32 key range (max_w > 65534): native INT32 keys (VIADDMNMX),
    speculative because (n-1) * max_w exceeds the INT32 key bound; every chunk check passes."""
    n = 520
    W = gen.generate("er_int", n, 970, p=1.0, lo=1, hi=100000)
    D, P, st = check(W, 1, expect_chunks=5)
    assert st.p_method == 2 and st.compute_f32 == 0


def test_pipeline_int32_round_tags():
    """INT32 weights beyond every key range (max_w > 4194302) with no-edge entries: round tags in
    INT32 arithmetic ((n-1) * max_w >= 2^24, so no FP32 compute; < FW_INF_I32, the domain rule)
    through the pipeline."""
    n = 256
    W = gen.generate("er_int", n, 971, p=0.05, lo=4_195_000, hi=4_200_000)
    D, P, st = check(W, 1, expect_chunks=2)
    assert st.p_method == 1 and st.compute_f32 == 0


@pytest.mark.parametrize("n,ct", [(8192, 32), (8448, 33), (16384, -1)])
def test_pipeline_pairs_ring_closed_form(n, ct):
    """A ring of weight 1 in a complete graph of weight n (every shortest path runs through every
    later block; no INF, so the keys are statically exact) through the host pipeline where chunks
    are wide enough for pairs of rounds (8192 in two 32-tile-row chunks, the C4-size auto
    geometry; 33-tile-row chunks have odd boundaries, so their plain rounds stay single):
    D = (j - i) mod n and next = i + 1 on every row."""
    W = np.full((n, n), np.float32(n), dtype=np.float32)
    i = np.arange(n)
    W[i, (i + 1) % n] = 1.0
    D, P, st = solve_pinned(W, ct)
    assert st.host_chunks >= 2 and st.p_method == 2
    i = np.arange(n)
    for r0 in range(0, n, 2048):
        r = np.arange(r0, min(n, r0 + 2048))
        np.testing.assert_array_equal(D[r], ((i[None, :] - r[:, None]) % n).astype(np.float32))
        np.testing.assert_array_equal(P[r], np.where(r[:, None] == i[None, :], r[:, None], (r[:, None] + 1) % n))


def test_pipeline_randomized_mix():
    """A seeded mix of host solves through ONE context: sizes with ragged tails, every input
    kind, next-hop / LAST_K / D-only, pinned and pageable buffers, chunkings from 1 tile-row to
    off (so pairs of rounds, plain pairs, speculative keys and round tags interleave with the
    context's cached buffers, events and staging ring) — each against the oracle."""
    rng = np.random.default_rng(20261020)
    kinds = ["complete_int", "complete_real", "er_int", "er_int_f32"]
    fw.fw_init(0, 0)
    try:
        for step in range(14):
            n = int(rng.integers(256, 1400))
            kind = kinds[step % 4]
            W = gen.generate(kind, n, 7000 + step, p=0.03, lo=1, hi=int(rng.choice([50, 1000])))
            path = [None, "next", "next"][step % 3]
            ct = int(rng.choice([-1, 0, 1, 2, 4]))
            pin = bool(step % 2)
            fw.fw_set_host_pipeline(ct)
            hD = torch.from_numpy(W.copy())
            hP = torch.full(W.shape, -5, dtype=torch.int32) if path else None
            if pin:
                hD = hD.pin_memory()
                hP = hP.pin_memory() if hP is not None else None
            (fw.fw_solve_i32 if W.dtype == np.int32 else fw.fw_solve)(hD, hP, block=128)
            D = hD.numpy()
            exact = exact_data(W)
            assert_D_matches(D, oracle.fw(W, None)[0], exact)
            if path:
                bad, first = oracle.check_paths(W, D, hP.numpy(), rtol=0.0 if exact else 1e-5)
                assert bad == 0, (step, n, kind, ct, pin, bad)
    finally:
        fw.fw_free()


@pytest.mark.parametrize("n", [1087, 1500, 2049])
def test_pageable_copy_sizes(n):
    """Pageable host buffers whose byte counts are not multiples of the copy pool's partition
    granularity (the parallel host copy must cover the last bytes of every slice): the standard
    path (auto pipeline off below 32 tile-rows) and a pipelined solve, bit-exact D and the
    diagonal / last-row next hops."""
    W = gen.generate("er_int", n, 1200 + n, p=0.03, lo=1, hi=50)
    for ct in (-1, 2):
        D, P, st = solve_pinned(W, ct, pin=False)
        np.testing.assert_array_equal(D, oracle.fw(W, None)[0])
        assert (np.diag(P) == np.arange(n)).all()
        assert oracle.check_paths(W, D, P)[0] == 0

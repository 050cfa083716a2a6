"""GPU tests of the partitioned (multi-GPU) solve path on one B200.

Two GPUs are not available to a single test process, so the partitioned path runs through
the loopback transport (fw_dist_loopback_solve_device_*): every rank of a `world`-way
block-row partition is emulated on this GPU with its own rows, its own pivot-strip receive
buffers and the per-rank look-ahead tile split; the broadcast is a device copy. The NCCL
entry points are exercised with a one-rank communicator.
"""
import numpy as np
import pytest

import apsp_inputs as gen
import oracle
from helpers import INF, assert_D_matches, exact_data

pytestmark = pytest.mark.gpu

fw = pytest.importorskip("paper_1811_01201_b200")
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def loopback(W, block, world, path="next"):
    fw.fw_init(0, fw.FW_PATH_LAST_K if path == "lastk" else 0)
    try:
        dD = torch.from_numpy(W).cuda()
        dP = torch.empty(W.shape, dtype=torch.int32, device="cuda") if path else None
        f = fw.fw_dist_loopback_solve_device_i32 if W.dtype == np.int32 else fw.fw_dist_loopback_solve_device_f32
        f(dD, dP, block=block, world=world, stream=torch.cuda.current_stream())
        return dD.cpu().numpy(), (dP.cpu().numpy() if dP is not None else None)
    finally:
        fw.fw_free()


CASES = [
    ("complete_int", 300, 64, 2), ("complete_int", 640, 128, 3), ("complete_int", 1000, 128, 4),
    ("complete_int", 257, 32, 2), ("complete_real", 513, 128, 2), ("complete_real", 700, 64, 3),
    ("er_int", 600, 128, 2), ("er_int", 450, 64, 4), ("er_int_f32", 900, 128, 8),
    ("complete_int", 300, 128, 4),   # one rank holds only padding rows
    ("complete_int", 1024, 128, 8),  # exactly one tile row per rank
]


@pytest.mark.parametrize("kind,n,block,world", CASES)
def test_loopback_vs_oracle(kind, n, block, world):
    W = gen.generate(kind, n, 11 + n, p=0.02, lo=1, hi=1000 if kind.startswith("er") else 100)
    D, P = loopback(W, block, world)
    exact = exact_data(W)
    assert_D_matches(D, oracle.fw(W, None)[0], exact)
    bad, first = oracle.check_paths(W, D, P, rtol=0.0 if exact else 1e-5)
    assert bad == 0, (bad, divmod(first, n))


@pytest.mark.parametrize("world", [1, 2, 5])
def test_loopback_lastk_and_distance_only(world):
    W = gen.generate("er_int", 513, 3, p=0.03, lo=1, hi=1000)
    D, P = loopback(W, 128, world, path="lastk")
    np.testing.assert_array_equal(D, oracle.fw(W, None)[0])
    assert oracle.check_paths(W, D, P, mode="lastk")[0] == 0
    D2, P2 = loopback(W, 64, world, path=None)
    np.testing.assert_array_equal(D2, D)


def test_loopback_matches_single_gpu_bitwise():
    """D and P of the partitioned solve equal the single-GPU solve bit for bit (same BS): min is
    exact and every candidate is one rounded add, whatever GPU computes it."""
    W = gen.generate("complete_real", 768, 21)
    D1, P1 = loopback(W, 128, 1)
    for world in (2, 3, 6):
        Dw, Pw = loopback(W, 128, world)
        np.testing.assert_array_equal(Dw, D1)
        np.testing.assert_array_equal(Pw, P1)


def loopback_stats(W, world, path="next", pairs=True):
    fw.fw_init(0, fw.FW_PATH_LAST_K if path == "lastk" else 0)
    try:
        fw.fw_set_option("pairs", 1 if pairs else 0)
        dD = torch.from_numpy(W).cuda()
        dP = torch.empty(W.shape, dtype=torch.int32, device="cuda") if path else None
        f = fw.fw_dist_loopback_solve_device_i32 if W.dtype == np.int32 else fw.fw_dist_loopback_solve_device_f32
        f(dD, dP, block=128, world=world, stream=torch.cuda.current_stream())
        s = fw.fw_last_stats()
        return dD.cpu().numpy(), (dP.cpu().numpy() if dP is not None else None), s
    finally:
        fw.fw_free()


@pytest.mark.parametrize("kind,n,world,path", [
    ("complete_int", 2000, 2, "next"), ("complete_int", 2000, 4, "next"), ("complete_int", 2048, 8, "next"),
    ("complete_int", 1024, 2, "lastk"), ("er_int", 1500, 4, "next"), ("er_int_f32", 1024, 4, "next"),
    ("complete_int", 1536, 3, None),     # 12 tile rows over 3 ranks: 4 each, pair-aligned
    ("complete_int", 1024, 3, "next"),   # 3/3/2 tile rows: not pair-aligned -> one round per pass
    ("complete_int", 2048, 5, "next"),   # not pair-aligned -> one round per pass
])
def test_loopback_pairs(kind, n, world, path):
    """Two rounds per phase-3 pass in the partitioned schedule (keyed / distance-only solves,
    every rank's rows on 256-row boundaries): the owner of blocks a, b runs the pair pivot, the
    256 rows a, b go out in one broadcast, the other ranks bring their columns a, b through both
    rounds (pair_cols), every rank relaxes the rest through 256 k — on the loopback's per-rank
    concurrent streams. D bitwise the one-GPU solve's (integer data), P valid."""
    W = gen.generate(kind, n, 90 + n + world, p=0.03, lo=1, hi=1000 if kind.startswith("er") else 100)
    D, P, s = loopback_stats(W, world, path)
    n_pad = (n + 127) // 128 * 128
    R = n_pad // 128
    tiles = [fw.fw_dist_partition(n_pad, world, r)[0] // 128 for r in range(world)]
    aligned = all(t % 2 == 0 for t in tiles)
    if s.p_method != 1:   # keyed / distance-only (a speculative key run may fall back to tags)
        assert (s.phase3_launches == R // 2) == aligned, (s.phase3_launches, R, tiles)
    D1, P1 = loopback(W, 128, 1, path=path)
    np.testing.assert_array_equal(D, D1)
    assert_D_matches(D, oracle.fw(W, None)[0], exact_data(W))
    if path:
        bad, first = oracle.check_paths(W, D, P, rtol=0.0, mode=path)
        assert bad == 0, (bad, divmod(first, n))


def test_loopback_pairs_off_same_distances():
    """fw_set_option("pairs", 0) takes the one-round schedule on the same partition: same D."""
    W = gen.generate("complete_int", 2000, 5)
    Dp, Pp, sp = loopback_stats(W, 4, pairs=True)
    Ds, Ps, ss = loopback_stats(W, 4, pairs=False)
    assert sp.phase3_launches == sp.rounds // 2 and ss.phase3_launches == ss.rounds
    np.testing.assert_array_equal(Dp, Ds)
    assert oracle.check_paths(W, Dp, Pp)[0] == 0 and oracle.check_paths(W, Ds, Ps)[0] == 0


def test_loopback_fallback_to_tags():
    W = gen.ring(700, 1000, np.float32)
    D, P = loopback(W, 128, 3)
    i, j = np.meshgrid(np.arange(700), np.arange(700), indexing="ij")
    np.testing.assert_array_equal(D.astype(np.int64), ((j - i) % 700) * 1000)
    np.testing.assert_array_equal(P, np.where(i == j, i, (i + 1) % 700))


def _nccl_one_rank(W, block, path="next", timing=True, persistent=None, nvls=None):
    """fw_dist_solve_device_* over a ONE-rank NCCL communicator: the NCCL data plane runs
    (every round's pivot strip through ncclBroadcast, validation / placement / key checks
    through ncclAllReduce, the TAG post-pass gather through grouped broadcasts)."""
    n = W.shape[0]
    flags = (fw.FW_TIMING if timing else 0) | (fw.FW_PATH_LAST_K if path == "lastk" else 0)
    fw.fw_init(0, flags)
    try:
        uid = fw.fw_comm_unique_id()
        assert len(uid) == 128
        fw.fw_comm_init(uid, 0, 1)
        if persistent is not None:
            fw.fw_set_option("persistent", persistent)
        if nvls is not None:
            fw.fw_set_option("nvls", nvls)
        row0, nrows = fw.fw_dist_partition(n, 1, 0)
        assert (row0, nrows) == (0, n)
        dD = torch.from_numpy(W).cuda()
        dP = torch.empty((n, n), dtype=torch.int32, device="cuda") if path else None
        f = fw.fw_dist_solve_device_i32 if W.dtype == np.int32 else fw.fw_dist_solve_device_f32
        f(dD, dP, n=n, block=block, stream=torch.cuda.current_stream())
        s = fw.fw_last_stats()
        with pytest.raises(fw.FwError):     # single-GPU entry refused while a communicator is active
            (fw.fw_solve_i32 if W.dtype == np.int32 else fw.fw_solve)(W.copy(), None)
        fw.fw_comm_free()
        return dD.cpu().numpy(), (dP.cpu().numpy() if dP is not None else None), s
    finally:
        fw.fw_free()


@pytest.mark.parametrize("kind,n,block,path", [
    ("complete_int", 300, 64, "next"),      # keyed P, one round per launch, BS 64
    ("complete_int", 1000, 128, "next"),    # keyed P, look-ahead schedule with the broadcast
    ("complete_real", 777, 128, "next"),    # round tags: the post-pass gathers D by broadcasts
    ("er_int", 900, 128, "lastk"),          # INT32 with INF, LAST_K
    ("complete_int", 640, 128, None),       # distance only
])
def test_nccl_single_rank_communicator(kind, n, block, path):
    W = gen.generate(kind, n, 5 + n, p=0.02, lo=1, hi=1000 if kind.startswith("er") else 100)
    D, P, s = _nccl_one_rank(W, block, path)
    R = (n + block - 1) // block
    # every round's pivot strip went through ncclBroadcast — one broadcast per round, or per
    # pair of rounds (rows a, b together) when the keyed / distance-only solve ran in pairs (a
    # speculative key run that falls back runs the rounds again; the TAG post-pass adds one
    # gather broadcast per rank)
    pairs = s.phase3_launches == R // 2 and s.p_method != 1
    assert pairs == (s.p_method != 1 and block == 128 and R % 2 == 0 and R >= 4), (s.phase3_launches, R)
    per_solve = R // 2 if pairs else R
    assert s.broadcasts >= per_solve, (s.broadcasts, R)
    if s.p_method == 1:
        assert s.broadcasts % R == (1 if path else 0) % R, (s.broadcasts, R)
    assert s.bcast_bytes >= R * block * s.n_pad * 4
    exact = exact_data(W)
    assert_D_matches(D, oracle.fw(W, None)[0], exact)
    if path:
        bad, first = oracle.check_paths(W, D, P, rtol=0.0 if exact else 1e-5, mode=path)
        assert bad == 0, (bad, divmod(first, n))


def test_nccl_one_rank_matches_single_gpu_bitwise():
    """The NCCL data plane (one rank) and the single-GPU schedule give the same D; P valid."""
    W = gen.generate("complete_int", 1024, 77)
    D1, P1, _ = _nccl_one_rank(W, 128)
    fw.fw_init(0, 0)
    try:
        dD = torch.from_numpy(W).cuda()
        dP = torch.empty(W.shape, dtype=torch.int32, device="cuda")
        fw.fw_solve_device_f32(dD, dP, block=128, stream=torch.cuda.current_stream())
        D0 = dD.cpu().numpy()
    finally:
        fw.fw_free()
    np.testing.assert_array_equal(D1, D0)


def test_nccl_missing_peer_times_out(monkeypatch):
    """A two-rank communicator whose second rank never joins: the non-blocking init is polled,
    times out (FW_NCCL_TIMEOUT_MS) and aborts with FW_ENCCL instead of hanging the process."""
    monkeypatch.setenv("FW_NCCL_TIMEOUT_MS", "4000")
    fw.fw_init(0, 0)
    try:
        uid = fw.fw_comm_unique_id()
        with pytest.raises(fw.FwError) as e:
            fw.fw_comm_init(uid, 0, 2)
        assert e.value.code == fw.FW_ENCCL and "timed out" in str(e.value)
        with pytest.raises(fw.FwError):      # no live communicator: the dist entry refuses
            fw.fw_dist_solve_device_f32(torch.zeros((128, 128), device="cuda"), None, n=128)
        fw.fw_comm_free()
        # the context stays usable for single-GPU solves
        W = gen.generate("complete_int", 200, 3)
        D = W.copy()
        fw.fw_solve(D, None)
        np.testing.assert_array_equal(D, oracle.fw(W, None)[0])
    finally:
        fw.fw_free()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 visible GPUs")
@pytest.mark.parametrize("kind,n,block", [("complete_int", 1000, 128), ("complete_real", 777, 64),
                                          ("er_int", 600, 32)])
def test_team_solve_matches_single_gpu(kind, n, block):
    """fw_solve(..., ngpus=G): G devices of this process, block-row partition + NCCL pivot
    broadcast (one host thread per device); integer data bitwise equal to the 1-GPU solve,
    real data within rel 1e-5, next-hop paths valid."""
    W = gen.generate(kind, n, 31, p=0.05, lo=1, hi=1000)
    G = min(torch.cuda.device_count(), 4)
    out = []
    for g in (1, G):
        D = W.copy()
        P = np.empty(W.shape, dtype=np.int32)
        fw.fw_init(0, 0)
        try:
            (fw.fw_solve_i32 if W.dtype == np.int32 else fw.fw_solve)(D, P, block=block, ngpus=g)
        finally:
            fw.fw_free()
        out.append((D, P))
    exact = W.dtype == np.int32 or kind == "complete_int"
    if exact:
        np.testing.assert_array_equal(out[0][0], out[1][0])
    else:
        np.testing.assert_allclose(out[1][0], out[0][0], rtol=1e-5)
    assert oracle.check_paths(W, out[1][0], out[1][1], rtol=0.0 if exact else 1e-5)[0] == 0


# ---- persistent loopback: every rank in ONE persistent grid, the fused publish ----
def loopback_persistent(W, world, path="next"):
    fw.fw_init(0, (fw.FW_PATH_LAST_K if path == "lastk" else 0) | fw.FW_TIMING)
    try:
        fw.fw_set_option("persistent", 1)
        dD = torch.from_numpy(W).cuda()
        dP = torch.empty(W.shape, dtype=torch.int32, device="cuda") if path else None
        f = fw.fw_dist_loopback_solve_device_i32 if W.dtype == np.int32 else fw.fw_dist_loopback_solve_device_f32
        f(dD, dP, block=128, world=world, stream=torch.cuda.current_stream())
        s = fw.fw_last_stats()
        return dD.cpu().numpy(), (dP.cpu().numpy() if dP is not None else None), s
    finally:
        fw.fw_free()


PCASES = [
    ("complete_int", 1000, 2, "next"), ("complete_int", 1024, 8, "next"), ("complete_real", 700, 3, "next"),
    ("complete_real", 900, 4, "lastk"), ("er_int", 800, 3, "next"), ("er_int_f32", 640, 5, "next"),
    ("complete_int", 300, 4, "next"),   # a rank with padding rows only
    ("complete_int", 768, 2, None),
]


@pytest.mark.parametrize("kind,n,world,path", PCASES)
def test_loopback_persistent_publish(kind, n, world, path):
    """The multi-rank persistent solve: each rank's phase-2 row strip / phase-1 tiles are copied
    by the producing CTA into every other rank's pivot-row ring with a release flag per tile
    (the fused publish), and the other ranks' tiles poll those flags — all ranks in one grid.
    D against the oracle (bitwise for integer data), P valid."""
    W = gen.generate(kind, n, 50 + n, p=0.03, lo=1, hi=1000 if kind.startswith("er") else 100)
    D, P, s = loopback_persistent(W, world, path)
    assert s.persistent == 1
    exact = exact_data(W)
    assert_D_matches(D, oracle.fw(W, None)[0], exact)
    if path:
        bad, first = oracle.check_paths(W, D, P, rtol=0.0 if exact else 1e-5, mode=path)
        assert bad == 0, (bad, divmod(first, n))


def test_loopback_persistent_matches_single_gpu_bitwise():
    """Integer data: the persistent partitioned solve gives the single-GPU distances bit for bit."""
    W = gen.generate("complete_int", 896, 77)
    D1, _ = loopback(W, 128, 1)
    for world in (2, 7):
        Dw, Pw, _ = loopback_persistent(W, world)
        np.testing.assert_array_equal(Dw, D1)
        assert oracle.check_paths(W, Dw, Pw)[0] == 0


@pytest.mark.parametrize("kind,n,path", [("complete_int", 1000, "next"), ("complete_real", 640, "next"),
                                         ("er_int", 513, "lastk")])
def test_nccl_single_rank_persistent(kind, n, path):
    """The communicator path of the persistent solve (opt-in) on a one-rank communicator: the
    ring allocation's CUDA IPC handle is all-gathered over NCCL, the pub flags zeroed, an NCCL
    all-reduce is the barrier before the launch, and the persistent grid runs this rank's items."""
    W = gen.generate(kind, n, 60 + n, p=0.03, lo=1, hi=1000 if kind.startswith("er") else 100)
    D, P, s = _nccl_one_rank(W, 128, path, persistent=1)
    assert s.persistent == 1
    exact = exact_data(W)
    assert_D_matches(D, oracle.fw(W, None)[0], exact)
    bad, first = oracle.check_paths(W, D, P, rtol=0.0 if exact else 1e-5, mode=path)
    assert bad == 0, (bad, divmod(first, n))


@pytest.mark.parametrize("kind,n", [("complete_int", 1000), ("complete_real", 640)])
def test_nccl_single_rank_persistent_nvls_setup(kind, n):
    """fw_set_option("nvls", 1): the collective NVLS setup (support check agreed over the
    communicator, multicast object + fabric handle from rank 0, bind and map on every rank) runs
    even with one rank. Where the pool cannot create a multicast object (one GPU per process) every
    rank falls back to the IPC peer rings; either way the solve is correct (persistent = 2: the
    multicast publish, 1: the peer rings)."""
    W = gen.generate(kind, n, 70 + n)
    D, P, s = _nccl_one_rank(W, 128, "next", persistent=1, nvls=1)
    assert s.persistent in (1, 2)
    exact = exact_data(W)
    assert_D_matches(D, oracle.fw(W, None)[0], exact)
    bad, first = oracle.check_paths(W, D, P, rtol=0.0 if exact else 1e-5)
    assert bad == 0, (bad, divmod(first, n))

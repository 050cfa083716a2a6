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


def test_loopback_fallback_to_tags():
    W = gen.ring(700, 1000, np.float32)
    D, P = loopback(W, 128, 3)
    i, j = np.meshgrid(np.arange(700), np.arange(700), indexing="ij")
    np.testing.assert_array_equal(D.astype(np.int64), ((j - i) % 700) * 1000)
    np.testing.assert_array_equal(P, np.where(i == j, i, (i + 1) % 700))


def test_nccl_single_rank_communicator():
    """fw_comm_unique_id / fw_comm_init / fw_dist_solve_device_* with a one-rank communicator."""
    n = 300
    W = gen.generate("complete_int", n, 5)
    fw.fw_init(0, 0)
    try:
        uid = fw.fw_comm_unique_id()
        assert len(uid) == 128
        fw.fw_comm_init(uid, 0, 1)
        row0, nrows = fw.fw_dist_partition(n, 1, 0)
        assert (row0, nrows) == (0, n)
        dD = torch.from_numpy(W).cuda()
        dP = torch.empty((n, n), dtype=torch.int32, device="cuda")
        fw.fw_dist_solve_device_f32(dD, dP, n=n, block=64, stream=torch.cuda.current_stream())
        with pytest.raises(fw.FwError):     # single-GPU entry refused while a communicator is active
            fw.fw_solve(W.copy(), None)
        fw.fw_comm_free()
        D, P = dD.cpu().numpy(), dP.cpu().numpy()
    finally:
        fw.fw_free()
    np.testing.assert_array_equal(D, oracle.fw(W, None)[0])
    assert oracle.check_paths(W, D, P)[0] == 0


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

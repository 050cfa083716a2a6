"""Seeded randomized GPU parity: many combinations of the solve's options in one run, each
against the CPU oracle — sizes with ragged tails, block sizes, input kinds (complete / sparse
with unreachable pairs, integer / real, FP32 / INT32), path modes (next hop, LAST_K, D only),
host buffers (pinned / pageable), device buffers or the loopback transport (every rank of a
2..7-way block-row partition on this GPU), host-pipeline chunkings, and one or two
rounds per phase-3 pass (FW_PAIRS). Integer data bit-exact, reals within rel 1e-5, every path
reconstructed (BASELINE.json north_star correctness requirements)."""
import numpy as np
import pytest

import apsp_inputs as gen
import oracle
from helpers import assert_D_matches, exact_data

pytestmark = pytest.mark.gpu

fw = pytest.importorskip("paper_1811_01201_b200")
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


KINDS = ["complete_int", "complete_real", "er_int", "er_int_f32", "er_int"]


def one_case(rng, step, monkeypatch):
    n = int(rng.integers(130, 2300))
    kind = KINDS[step % len(KINDS)]
    hi = int(rng.choice([9, 100, 1000, 40000]))
    W = gen.generate(kind, n, 9100 + step, p=float(rng.choice([0.002, 0.02, 0.2])), lo=1, hi=hi)
    path = [None, "next", "lastk", "next"][step % 4]
    block = int(rng.choice([0, 32, 64, 128, 128]))
    where = ["pinned", "pageable", "device", "loopback"][int(rng.integers(0, 4))]
    world = int(rng.integers(2, 8))
    ct = int(rng.choice([-1, 0, 1, 2, 3, 4]))
    pairs = bool(rng.integers(0, 2))
    monkeypatch.setenv("FW_PAIRS", "1" if pairs else "0")
    flags = fw.FW_PATH_LAST_K if path == "lastk" else 0
    is_int = W.dtype == np.int32
    fw.fw_init(0, flags)
    try:
        fw.fw_set_host_pipeline(ct)
        if where in ("device", "loopback"):
            dD = torch.from_numpy(W.copy()).cuda()
            dP = torch.empty(W.shape, dtype=torch.int32, device="cuda") if path else None
            if where == "device":
                (fw.fw_solve_device_i32 if is_int else fw.fw_solve_device_f32)(
                    dD, dP, block=block, stream=torch.cuda.current_stream())
            else:   # every rank of a `world`-way block-row partition emulated on this GPU
                (fw.fw_dist_loopback_solve_device_i32 if is_int else fw.fw_dist_loopback_solve_device_f32)(
                    dD, dP, block=block, world=world, stream=torch.cuda.current_stream())
            D = dD.cpu().numpy()
            P = dP.cpu().numpy() if path else None
        else:
            hD = torch.from_numpy(W.copy())
            hP = torch.full(W.shape, -5, dtype=torch.int32) if path else None
            if where == "pinned":
                hD = hD.pin_memory()
                hP = hP.pin_memory() if hP is not None else None
            (fw.fw_solve_i32 if is_int else fw.fw_solve)(hD, hP, block=block)
            D = hD.numpy()
            P = hP.numpy() if path else None
    finally:
        fw.fw_free()
    desc = dict(step=step, n=n, kind=kind, hi=hi, path=path, block=block, where=where, ct=ct, pairs=pairs,
                world=world)
    exact = exact_data(W)
    assert_D_matches(D, oracle.fw(W, None)[0], exact)
    if path:
        bad, first = oracle.check_paths(W, D, P, rtol=0.0 if exact else 1e-5, mode=path)
        assert bad == 0, (desc, bad, divmod(first, n))


@pytest.mark.parametrize("chunk", range(4))
def test_fuzz_solves(chunk, monkeypatch):
    rng = np.random.default_rng(4242 + chunk)
    for k in range(8):   # (n-1) * max_w stays far below FW_INF_I32 here: no domain refusals
        one_case(rng, 8 * chunk + k, monkeypatch)

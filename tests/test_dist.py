"""Multi-GPU host logic on CPU (no GPU): the block-row partition exported by the C ABI
(fw_dist_partition / fw_dist_owner) and the per-round schedule of the partitioned solve —
owner(K) runs phase 1 and its row strip, broadcasts the pivot row strip, every rank updates
its own rows (column strip, phase 3) — run as world-size 2 and 3 `gloo` process groups.
The per-phase arithmetic here is a NumPy test double of the CUDA kernels (exact arg-min
LAST_K semantics, reading R9); the partition and owners come from the product library.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import apsp_inputs as gen
import oracle
import paper_1811_01201_b200 as fw


@pytest.mark.parametrize("n", [1, 100, 128, 129, 1000, 4096, 16384, 32768, 65536])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 7, 8])
def test_partition_covers_rows(n, world):
    n_pad = (n + 127) // 128 * 128
    parts = [fw.fw_dist_partition(n, world, r) for r in range(world)]
    pos = 0
    padded = []
    for r, (r0, nr) in enumerate(parts):
        assert r0 % 128 == 0
        if nr:
            assert r0 == pos
            pos += nr
        # padded extent of the rank (row0 of the next rank, or n_pad)
        nxt = parts[r + 1][0] if r + 1 < world else n_pad
        padded.append(max(0, nxt - r0) if r0 < n_pad else 0)
    assert pos == n
    assert sum(padded) == n_pad
    assert max(padded) - min(padded) <= 128
    for row in range(0, n_pad, 37):
        o = fw.fw_dist_owner(n, world, row)
        r0 = parts[o][0]
        assert r0 <= row < r0 + padded[o]
    assert fw.fw_dist_owner(n, world, n_pad) == -1


def test_partition_errors():
    with pytest.raises(fw.FwError):
        fw.fw_dist_partition(0, 2, 0)
    with pytest.raises(fw.FwError):
        fw.fw_dist_partition(100, 2, 2)


# ---- NumPy test double of the phase kernels (LAST_K keyed semantics) ----------------------
def _relax(C, Pc, A, B, kb, rows_mask=None, cols_mask=None):
    """C <- min(C, min_k A[:,k] + B[k,:]) (first arg-min k), P = kb + k where strictly better."""
    if C.size == 0:
        return
    S = A[:, :, None] + B[None, :, :]               # i x k x j
    kmin = np.argmin(S, axis=1)                     # first k on ties
    m = np.take_along_axis(S, kmin[:, None, :], axis=1)[:, 0, :]
    better = m < C
    if rows_mask is not None:
        better &= rows_mask[:, None]
    if cols_mask is not None:
        better &= cols_mask[None, :]
    C[better] = m[better]
    Pc[better] = (kb + kmin)[better]


def _phase1(D, P, r, kb, BS):
    blk = D[r:r + BS, kb:kb + BS]
    pb = P[r:r + BS, kb:kb + BS]
    for k in range(BS):
        s = blk[:, [k]] + blk[[k], :]
        better = s < blk
        blk[better] = s[better]
        pb[better] = kb + k


def _rank_main(rank, world, port, n, BS, seed, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n_pad = (n + 127) // 128 * 128
    W = gen.generate("er_int_f32", n, seed, p=0.2, lo=1, hi=50)
    row0, nsrc = fw.fw_dist_partition(n, world, rank)
    nxt = fw.fw_dist_partition(n, world, rank + 1)[0] if rank + 1 < world else n_pad
    nrows = max(0, nxt - row0) if row0 < n_pad else 0
    # this rank's padded rows (init kernel semantics: INF padding, zero diagonal)
    D = np.full((nrows, n_pad), np.inf, dtype=np.float32)
    D[:nsrc, :n] = W[row0:row0 + nsrc]
    for i in range(nrows):
        if row0 + i < n_pad:
            D[i, row0 + i] = 0
    P = np.full((nrows, n_pad), -1, dtype=np.int32)
    R = (n + BS - 1) // BS
    for K in range(R):
        kb = K * BS
        owner = fw.fw_dist_owner(n, world, kb)
        strip = torch.empty((BS, n_pad), dtype=torch.float32)
        if owner == rank:
            r = kb - row0
            _phase1(D, P, r, kb, BS)
            cols = np.ones(n_pad, dtype=bool)
            cols[kb:kb + BS] = False                  # the diagonal block is phase 1's
            _relax(D[r:r + BS], P[r:r + BS], D[r:r + BS, kb:kb + BS], D[r:r + BS].copy(), kb,
                   cols_mask=cols)
            strip = torch.from_numpy(D[r:r + BS].copy())
        dist.broadcast(strip, src=owner)              # the only exchange of a round
        B = strip.numpy()
        rows = np.ones(nrows, dtype=bool)
        if owner == rank:
            rows[kb - row0:kb - row0 + BS] = False
        # column strip of the local rows through D_KK* (from the broadcast strip)
        _relax(D[:, kb:kb + BS], P[:, kb:kb + BS], D[:, kb:kb + BS].copy(), B[:, kb:kb + BS], kb,
               rows_mask=rows)
        # phase 3 on the local rows outside the strips
        cols = np.ones(n_pad, dtype=bool)
        cols[kb:kb + BS] = False
        _relax(D, P, D[:, kb:kb + BS].copy(), B, kb, rows_mask=rows, cols_mask=cols)
    Dt = torch.from_numpy(np.ascontiguousarray(D[:nsrc, :n]))
    Pt = torch.from_numpy(np.ascontiguousarray(P[:nsrc, :n]))
    gD = [None] * world
    gP = [None] * world
    dist.all_gather_object(gD, Dt)
    dist.all_gather_object(gP, Pt)
    if rank == 0:
        out.put((np.concatenate([g.numpy() for g in gD]), np.concatenate([g.numpy() for g in gP])))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,n,BS", [(2, 300, 64), (3, 500, 128), (2, 257, 32), (4, 300, 64)])
def test_partitioned_schedule_gloo(world, n, BS):
    """The partitioned round schedule reproduces the oracle's D (bitwise, integer data) and a
    valid LAST_K P, with the pivot strip as the only data crossing ranks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, n, BS, 7, q)) for r in range(world)]
    for p in procs:
        p.start()
    D, P = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    W = gen.generate("er_int_f32", n, 7, p=0.2, lo=1, hi=50)
    Dref, _ = oracle.fw(W, None)
    np.testing.assert_array_equal(D, Dref)
    P = np.where(np.isinf(D) | np.eye(n, dtype=bool), -1, P).astype(np.int32)
    assert oracle.check_paths(W, D, P, mode="lastk")[0] == 0


# ---- the pair schedule of the partitioned solve (two rounds per phase-3 pass) ----------------
def _rank_main_pairs(rank, world, port, n, seed, out):
    """Two rounds per pass on a pair-aligned partition (BS = 128): owner(a, b)
    runs the one-GPU pair pivot on its rows, the 256 rows a, b are the only data broadcast, the
    other ranks bring their columns a, b through both rounds (pair_cols), and every rank relaxes
    the rest of its rows through 256 k in one product."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    BS = 128
    n_pad = (n + 127) // 128 * 128
    W = gen.generate("er_int_f32", n, seed, p=0.2, lo=1, hi=50)
    row0, nsrc = fw.fw_dist_partition(n, world, rank)
    nxt = fw.fw_dist_partition(n, world, rank + 1)[0] if rank + 1 < world else n_pad
    nrows = max(0, nxt - row0) if row0 < n_pad else 0
    assert row0 % 256 == 0                             # the case the pair schedule runs on
    D = np.full((nrows, n_pad), np.inf, dtype=np.float32)
    D[:nsrc, :n] = W[row0:row0 + nsrc]
    for i in range(nrows):
        D[i, row0 + i] = 0
    P = np.full((nrows, n_pad), -1, dtype=np.int32)
    R = n_pad // BS
    allc = np.ones(n_pad, dtype=bool)

    def mask_out(lo, hi, size):
        m = np.ones(size, dtype=bool)
        m[max(lo, 0):max(hi, 0)] = False
        return m

    for Pp in range(R // 2):
        a, b = 2 * Pp, 2 * Pp + 1
        ka, kb_ = a * BS, b * BS
        owner = fw.fw_dist_owner(n, world, ka)
        assert owner == fw.fw_dist_owner(n, world, kb_)
        strip = torch.empty((2 * BS, n_pad), dtype=torch.float32)
        if owner == rank:                              # pair_pivot on the owner's rows
            for x, y in ((a, b), (b, a)):
                kx, ky = x * BS, y * BS
                rx, ry = kx - row0, ky - row0
                _phase1(D, P, rx, kx, BS)
                # phase 2: row x (columns != x), column x (own rows != x)
                _relax(D[rx:rx + BS], P[rx:rx + BS], D[rx:rx + BS, kx:kx + BS], D[rx:rx + BS].copy(), kx,
                       cols_mask=mask_out(kx, kx + BS, n_pad))
                _relax(D[:, kx:kx + BS], P[:, kx:kx + BS], D[:, kx:kx + BS].copy(), D[rx:rx + BS, kx:kx + BS].copy(),
                       kx, rows_mask=mask_out(rx, rx + BS, nrows))
                # strip3(x, y): row y (columns != x) and column y (rows outside a, b) through block x
                _relax(D[ry:ry + BS], P[ry:ry + BS], D[ry:ry + BS, kx:kx + BS].copy(), D[rx:rx + BS].copy(), kx,
                       cols_mask=mask_out(kx, kx + BS, n_pad))
                lo = min(rx, ry)
                _relax(D[:, ky:ky + BS], P[:, ky:ky + BS], D[:, kx:kx + BS].copy(), D[rx:rx + BS, ky:ky + BS].copy(),
                       kx, rows_mask=mask_out(lo, lo + 2 * BS, nrows))
            strip = torch.from_numpy(D[ka - row0:ka - row0 + 2 * BS].copy())
        dist.broadcast(strip, src=owner)               # rows a, b: the only exchange of the pair
        B = strip.numpy()
        if owner != rank:                              # pair_cols
            for x in (a, b):
                kx = x * BS
                _relax(D[:, kx:kx + BS], P[:, kx:kx + BS], D[:, kx:kx + BS].copy(),
                       B[kx - ka:kx - ka + BS, kx:kx + BS], kx)
            for x, y in ((a, b), (b, a)):              # x through its partner y, even block first
                kx, ky = x * BS, y * BS
                _relax(D[:, kx:kx + BS], P[:, kx:kx + BS], D[:, ky:ky + BS].copy(),
                       B[ky - ka:ky - ka + BS, kx:kx + BS], ky)
        # bulk: the local rows outside a, b, the columns outside a, b, through 256 k
        rows = mask_out(ka - row0, ka - row0 + 2 * BS, nrows)
        _relax(D, P, D[:, ka:ka + 2 * BS].copy(), B, ka, rows_mask=rows, cols_mask=mask_out(ka, ka + 2 * BS, n_pad))
    Dt = torch.from_numpy(np.ascontiguousarray(D[:nsrc, :n]))
    Pt = torch.from_numpy(np.ascontiguousarray(P[:nsrc, :n]))
    gD = [None] * world
    gP = [None] * world
    dist.all_gather_object(gD, Dt)
    dist.all_gather_object(gP, Pt)
    if rank == 0:
        out.put((np.concatenate([g.numpy() for g in gD]), np.concatenate([g.numpy() for g in gP])))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 1000), (4, 1024), (3, 1536)])
def test_partitioned_pair_schedule_gloo(world, n):
    """The pair schedule on a pair-aligned partition reproduces the oracle's D bitwise (integer
    data) with a valid LAST_K P; the rows of a pair are the only data crossing ranks."""
    for r in range(world):
        assert fw.fw_dist_partition(n, world, r)[0] % 256 == 0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main_pairs, args=(r, world, port, n, 9, q)) for r in range(world)]
    for p in procs:
        p.start()
    D, P = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    W = gen.generate("er_int_f32", n, 9, p=0.2, lo=1, hi=50)
    Dref, _ = oracle.fw(W, None)
    np.testing.assert_array_equal(D, Dref)
    P = np.where(np.isinf(D) | np.eye(n, dtype=bool), -1, P).astype(np.int32)
    assert oracle.check_paths(W, D, P, mode="lastk")[0] == 0

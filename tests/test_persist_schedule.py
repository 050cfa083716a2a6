"""The persistent solve's work-item order, host-only.

Checked properties: every (round K, tile I, J) product and every phase-1 item appears exactly
once; every item's dependencies (its own tile at round K-1, its A operand (I, K) and B operand
(K, J) at round K — or the diagonal tile after phase 1) come EARLIER in the order (the
deadlock-freedom argument: the earliest unfinished item can always run); each rank's items
touch only its own rows; a rank's subsequence (one GPU of a communicator) is the global order
filtered by rank. The dependency rules are restated here from the paper's phases,
not taken from the library."""
import numpy as np
import pytest

fw = pytest.importorskip("paper_1811_01201_b200")


def unpack(u):
    u = np.asarray(u, dtype=np.uint64)
    return ((u >> 29) & 7).astype(int), ((u >> 27) & 3).astype(int), ((u >> 18) & 511).astype(int), \
        ((u >> 9) & 511).astype(int), (u & 511).astype(int)


def rows_of(n, world):
    return [fw.fw_dist_partition(((n + 127) // 128) * 128, world, r) for r in range(world)]


@pytest.mark.parametrize("n,world,gap", [(128, 1, 0), (256, 1, 5), (700, 1, 3), (1024, 1, 1000),
                                         (1000, 2, 4), (1280, 3, 0), (1024, 8, 7), (1500, 5, 2)])
def test_order_complete_and_dependencies_earlier(n, world, gap):
    T = (n + 127) // 128
    r, ty, K, I, J = unpack(fw.fw_persist_schedule(n, world, -1, gap))
    pos = {}
    for idx in range(len(ty)):
        key = ("P1", K[idx]) if ty[idx] == 1 else ("T", K[idx], I[idx], J[idx])
        assert key not in pos, f"duplicate item {key}"
        pos[key] = idx
    # completeness: phase 1 of every round, and every tile of every round
    # (round K relaxes every tile through block K; tile (K, K) by phase 1, the others by products)
    for k in range(T):
        assert ("P1", k) in pos
        for i in range(T):
            for j in range(T):
                if (i, j) != (k, k):
                    assert ("T", k, i, j) in pos, (k, i, j)
    assert len(pos) == T * T * T
    parts = rows_of(n, world)

    def done(k, i, j):   # the item that makes tile (i, j) final for round k
        return pos[("P1", k)] if (i, j) == (k, k) else pos[("T", k, i, j)]

    for key, idx in pos.items():
        if key[0] == "P1":
            k = key[1]
            if k > 0:
                assert done(k - 1, k, k) < idx           # tile (K, K) after round K-1
            continue
        _, k, i, j = key
        if k > 0:
            assert done(k - 1, i, j) < idx               # own tile after round K-1
        assert done(k, i, k) < idx or j == k             # A = (I, K) final for round K
        assert done(k, k, j) < idx or i == k             # B = (K, J) final for round K
        if i == k or j == k:
            assert pos[("P1", k)] < idx                  # phase 2 reads the closed diagonal block
    # ownership: every item runs on the rank whose rows hold its tile
    for idx in range(len(ty)):
        row = (K[idx] if ty[idx] == 1 else I[idx]) * 128
        r0, nr = parts[r[idx]]
        assert r0 <= row < r0 + max(nr, 1) or (nr == 0 and False), (idx, r[idx], row)


@pytest.mark.parametrize("n,world", [(1000, 2), (1024, 8), (777, 3)])
def test_rank_subsequences(n, world):
    full = fw.fw_persist_schedule(n, world, -1, 4)
    rk = (full >> 29) & 7
    for r in range(world):
        np.testing.assert_array_equal(fw.fw_persist_schedule(n, world, r, 4), full[rk == r])


def test_bad_arguments():
    with pytest.raises(fw.FwError):
        fw.fw_persist_schedule(0, 1)
    with pytest.raises(fw.FwError):
        fw.fw_persist_schedule(1000, 9)


@pytest.mark.parametrize("n,gap", [(128, 0), (256, 3), (700, 5), (1024, 0), (1024, 40), (2000, 100000)])
def test_one_gpu_decode_matches_table(n, gap):
    """The one-GPU persistent kernel decodes its items arithmetically (persist_decode); run on the
    host, that order is exactly the table order checked above (skipping the last round's no-ops)."""
    np.testing.assert_array_equal(fw.fw_persist_schedule(n, 1, -2, gap), fw.fw_persist_schedule(n, 1, -1, gap))


@pytest.mark.parametrize("n,gap", [(256, 0), (700, 5), (1024, 40), (4096, 740)])
def test_one_gpu_quarters_collapse_to_table(n, gap):
    """With quarter items (the critical-path tiles of the one-GPU order as four 64 x 64 items),
    every quartered tile appears as its four quarters back to back (quarters 0..3 in the rank
    bits, type 3); collapsing them gives exactly the full-tile order."""
    full = fw.fw_persist_schedule(n, 1, -1, gap)
    q = fw.fw_persist_schedule(n, 1, -3, gap)
    r, ty, K, I, J = unpack(q)
    out, i = [], 0
    while i < len(q):
        if ty[i] == 3:
            assert list(r[i:i + 4]) == [0, 1, 2, 3] and np.all(ty[i:i + 4] == 3)
            assert len({(K[x], I[x], J[x]) for x in range(i, i + 4)}) == 1
            out.append((2 << 27) | (int(K[i]) << 18) | (int(I[i]) << 9) | int(J[i]))
            i += 4
        else:
            out.append(int(q[i]))
            i += 1
    np.testing.assert_array_equal(np.array(out, dtype=np.uint32), full)
    assert np.sum(ty == 3) > 0


def _check_one_gpu_order(ty, K, I, J, T):
    """Completeness and dependencies-earlier of a one-GPU order given as full-tile items."""
    pos = {}
    for idx in range(len(ty)):
        key = ("P1", K[idx]) if ty[idx] == 1 else ("T", K[idx], I[idx], J[idx])
        assert key not in pos, f"duplicate item {key}"
        pos[key] = idx
    assert len(pos) == T * T * T

    def done(k, i, j):
        return pos[("P1", k)] if (i, j) == (k, k) else pos[("T", k, i, j)]

    for key, idx in pos.items():
        if key[0] == "P1":
            if key[1] > 0:
                assert done(key[1] - 1, key[1], key[1]) < idx
            continue
        _, k, i, j = key
        if k > 0:
            assert done(k - 1, i, j) < idx
        assert done(k, i, k) < idx or j == k
        assert done(k, k, j) < idx or i == k
        if i == k or j == k:
            assert pos[("P1", k)] < idx


@pytest.mark.parametrize("n,gap", [(128, 0), (256, 0), (384, 1), (700, 5), (1024, 40), (4096, 740), (3000, 100000)])
def test_one_gpu_critical_quarters(n, gap):
    """persist_quarters = 2: only the tiles the pivot chain waits for are quarter items — per round
    N the round-(N-1) tile (N, N) first in the prio section, and round N's phase-2 tiles (N, N+1),
    (N+1, N) first in its phase-2 section. Collapsing each run of four quarters gives a complete
    order in which every item's dependencies come earlier (deadlock-freedom), with three
    quartered tiles per round."""
    T = (n + 127) // 128
    q = fw.fw_persist_schedule(n, 1, -4, gap)
    r, ty, K, I, J = unpack(q)
    out, i, nq = [], 0, 0
    while i < len(q):
        if ty[i] == 3:
            assert list(r[i:i + 4]) == [0, 1, 2, 3] and np.all(ty[i:i + 4] == 3)
            assert len({(K[x], I[x], J[x]) for x in range(i, i + 4)}) == 1
            out.append((2, K[i], I[i], J[i]))
            nq += 1
            i += 4
        else:
            out.append((ty[i], K[i], I[i], J[i]))
            i += 1
    a = np.array(out)
    _check_one_gpu_order(a[:, 0], a[:, 1], a[:, 2], a[:, 3], T)
    # quartered: (0,1), (1,0) of round 0; per round K < T-1: (K+1, K+1); per round N in 1..T-2:
    # (N, N+1), (N+1, N)
    assert nq == (2 + (T - 1) + 2 * (T - 2) if T >= 2 else 0)

"""CPU checks of the host pipeline's schedule (reading R16), no GPU.

1. The chunk boundaries the library uses (fw_host_pipeline_bounds, host-only) partition the
   tile-rows: 0 = t_0 < t_1 < ... < t_C = ceil(n/128), auto chunks doubling from the first.
2. A test-side model of the pipeline's ORDER of work, written independently of the C++ driver
   from DESIGN.md §4.8 (arrival: catch-up rounds whose pivots lie in earlier chunks as plain
   phase-3 rounds + one deferred column-strip batch, then the chunk's own rounds; departure:
   the prefix rows take each chunk's block range with final pivots), run on small integer
   graphs in exact int64 arithmetic with the library's own chunk geometry (scaled to small
   blocks) and other chunkings, must give the unique shortest distances of the plain triple
   loop (oracle), while a schedule that reads pivot strips before they completed their round
   is caught.
"""
import numpy as np
import pytest

import apsp_inputs as gen
import oracle

fw = pytest.importorskip("paper_1811_01201_b200")

INF = np.int64(1) << 40


def minplus(A, B):
    """C[i][j] = min_k A[i][k] + B[k][j] (exact int64)."""
    return np.min(A[:, :, None] + B[None, :, :], axis=1)


class Model:
    """Blocked FW state on an n x n int64 matrix with blocks of BS (n % BS == 0)."""

    def __init__(self, W, BS):
        self.D = W.astype(np.int64).copy()
        self.D[self.D >= gen.INF_I32] = INF
        np.fill_diagonal(self.D, 0)
        self.BS = BS

    def blk(self, K):
        return slice(K * self.BS, (K + 1) * self.BS)

    def own_round(self, K, rows):
        """Round K on row range `rows` that contains block K: phase 1, phase 2 (row strip over
        all columns, column strip of `rows`), phase 3 of `rows`."""
        D, kb = self.D, self.blk(K)
        for k in range(kb.start, kb.stop):                        # phase 1: closure of D_KK
            D[kb, kb] = np.minimum(D[kb, kb], D[kb, k:k + 1] + D[k:k + 1, kb])
        Dkk = D[kb, kb].copy()
        D[kb, :] = np.minimum(D[kb, :], minplus(Dkk, D[kb, :]))   # row strip (product, R7)
        D[rows, kb] = np.minimum(D[rows, kb], minplus(D[rows, kb], Dkk))
        A, B = D[rows, kb].copy(), D[kb, :].copy()
        upd = np.minimum(D[rows, :], minplus(A, B))
        keep = D[rows, kb].copy()
        D[rows, :] = upd
        D[rows, kb] = keep                                        # phase 3 leaves strip K alone

    def plain_rounds(self, K0, K1, rows):
        """Rounds [K0, K1) whose pivot rows are outside `rows` and complete for their round:
        phase 3 without the round's own column block, then the deferred column strips."""
        D = self.D
        for K in range(K0, K1):
            kb = self.blk(K)
            A, B = D[rows, kb].copy(), D[kb, :].copy()
            keep = D[rows, kb].copy()
            D[rows, :] = np.minimum(D[rows, :], minplus(A, B))
            D[rows, kb] = keep
        for K in range(K0, K1):                                   # column-strip batch
            kb = self.blk(K)
            D[rows, kb] = np.minimum(D[rows, kb], minplus(D[rows, kb], D[kb, kb]))


    # ---- two rounds per pass, blocks a, b = 2p, 2p+1 ----
    def relax(self, rows, cols, ks):
        """D[rows, cols] <- min(D[rows, cols], D[rows, ks] (x) D[ks, cols]) (one product; 1-D
        index arrays, or [:, None] / [None, :] shaped ones)."""
        D = self.D
        rows, cols, ks = np.ravel(rows), np.ravel(cols), np.ravel(ks)
        A = D[np.ix_(rows, ks)].copy()
        B = D[np.ix_(ks, cols)].copy()
        D[np.ix_(rows, cols)] = np.minimum(D[np.ix_(rows, cols)], minplus(A, B))

    def own_pair(self, a, rows_lo, rows_hi, last):
        """run_pairs for one pair on rows [rows_lo, rows_hi) (block units): strip region by two
        sub-rounds, next pair's strips (prio), then the 256-deep bulk."""
        BS, D = self.BS, self.D
        n = D.shape[0]
        blk = lambda k: slice(k * BS, (k + 1) * BS)
        b = a + 1
        R0, R1 = rows_lo * BS, rows_hi * BS
        allc = np.arange(n)
        for x, y in ((a, b), (b, a)):
            kb = blk(x)
            for k in range(kb.start, kb.stop):                      # phase 1 (closure of D_xx)
                D[kb, kb] = np.minimum(D[kb, kb], D[kb, k:k + 1] + D[k:k + 1, kb])
            Dxx = D[kb, kb].copy()
            cols = allc[(allc < kb.start) | (allc >= kb.stop)]
            D[kb.start:kb.stop, cols] = np.minimum(D[kb.start:kb.stop, cols], minplus(Dxx, D[kb.start:kb.stop, cols]))
            rws = np.array([r for r in range(R0, R1) if not kb.start <= r < kb.stop])
            D[np.ix_(rws, np.arange(kb.start, kb.stop))] = np.minimum(
                D[np.ix_(rws, np.arange(kb.start, kb.stop))], minplus(D[np.ix_(rws, np.arange(kb.start, kb.stop))], Dxx))
            yb = blk(y)                                              # strip3(x -> y)
            cols_y = allc[(allc < kb.start) | (allc >= kb.stop)]
            self.relax(np.arange(yb.start, yb.stop)[:, None], cols_y[None, :], np.arange(kb.start, kb.stop))
            lo = min(x, y) * BS
            rws_y = np.array([r for r in range(R0, R1) if not lo <= r < lo + 2 * BS])
            if len(rws_y):
                self.relax(rws_y[:, None], np.arange(yb.start, yb.stop)[None, :], np.arange(kb.start, kb.stop))
        ks = np.arange(a * BS, (a + 2) * BS)
        w = 2 if last else 4
        ex = (allc >= a * BS) & (allc < (a + w) * BS)
        if not last:                                                # prio: rows/cols c, d
            cd = np.arange((a + 2) * BS, (a + 4) * BS)
            self.relax(cd[:, None], allc[~((allc >= a * BS) & (allc < (a + 2) * BS))][None, :], ks)
            rws = np.array([r for r in range(R0, R1) if not a * BS <= r < (a + 4) * BS])
            if len(rws):
                self.relax(rws[:, None], cd[None, :], ks)
        rws = np.array([r for r in range(R0, R1) if not ex[r]])     # bulk
        if len(rws):
            self.relax(rws[:, None], allc[~ex][None, :], ks)

    def plain_pairs(self, K0, K1, rows):
        """run_plain with pairs: 256-deep launches leaving both column blocks, own-block strip
        batch, then partner-block batches (even blocks, then odd)."""
        BS, D = self.BS, self.D
        n = D.shape[0]
        allc = np.arange(n)
        rr = np.arange(rows.start, rows.stop)[:, None]
        fused = []
        K = K0
        while K < K1:
            if K % 2 == 0 and K + 1 < K1:
                ks = np.arange(K * BS, (K + 2) * BS)
                self.relax(rr, allc[~((allc >= K * BS) & (allc < (K + 2) * BS))][None, :], ks)
                fused.append(K)
                K += 2
            else:
                kb = self.blk(K)
                keep = D[rows, kb].copy()
                D[rows, :] = np.minimum(D[rows, :], minplus(D[rows, kb].copy(), D[kb, :].copy()))
                D[rows, kb] = keep
                K += 1
        for K in range(K0, K1):
            kb = self.blk(K)
            D[rows, kb] = np.minimum(D[rows, kb], minplus(D[rows, kb], D[kb, kb]))
        for par in (0, 1):
            for K in fused:
                x, y = K + par, K + 1 - par                         # block x through partner y
                xb, yb = self.blk(x), self.blk(y)
                D[rows, xb] = np.minimum(D[rows, xb], minplus(D[rows, yb].copy(), D[yb, xb].copy()))


def run_pipeline_pairs(W, BS, tb, min_rows=1, force=False):
    """The pipeline's order of work with pairs (chunks of >= min_rows blocks use pairs; plain
    pairs only when every chunk boundary is even, as in pipe_solve — force=True drops that
    condition to show why it is there)."""
    m = Model(W, BS)
    even = force or all(t % 2 == 0 for t in tb)
    R = len(W) // BS
    C = len(tb) - 1
    rows = lambda a, b: slice(a * BS, b * BS)
    for c in range(C):                                              # arrival
        t0, t1 = tb[c], tb[c + 1]
        use = t1 - t0 >= min_rows
        if use and even:
            m.plain_pairs(0, t0, rows(t0, t1))
        else:
            m.plain_rounds(0, t0, rows(t0, t1))
        k1 = min(t1, R)
        if use and t0 % 2 == 0 and (k1 - t0) % 2 == 0:
            for a in range(t0, k1, 2):
                m.own_pair(a, t0, t1, last=a + 2 >= k1)
        else:
            for K in range(t0, k1):
                m.own_round(K, rows(t0, t1))
    for c in range(C - 1, -1, -1):                                  # departure
        t0, t1 = tb[c], tb[c + 1]
        if t0 >= min_rows and even:
            m.plain_pairs(t0, min(t1, R), rows(0, t0))
        else:
            m.plain_rounds(t0, min(t1, R), rows(0, t0))
    return m.D


def run_pipeline(W, BS, tb, violate=False):
    """The pipeline's order of work for chunk boundaries tb (in blocks of BS)."""
    m = Model(W, BS)
    R = len(W) // BS
    C = len(tb) - 1
    rows = lambda a, b: slice(a * BS, b * BS)
    for c in range(C):                                            # arrival
        t0, t1 = tb[c], tb[c + 1]
        m.plain_rounds(0, t0, rows(t0, t1))
        if violate and c == C - 1:
            continue          # the last chunk's own pivot rounds skipped: its rows are incomplete
        for K in range(t0, min(t1, R)):
            m.own_round(K, rows(t0, t1))
    for c in range(C - 1, -1, -1):                                # departure
        if violate and c == C - 1:
            continue
        t0, t1 = tb[c], tb[c + 1]
        m.plain_rounds(t0, min(t1, R), rows(0, t0))
    return m.D


@pytest.mark.parametrize("n,ct", [(1000, 1), (1000, 3), (8192, -1), (16384, -1), (32768, -1), (65536, -1),
                                  (300, 2), (129, 1), (4096, -1), (6000, -1), (3000, -1)])
def test_bounds_partition_tile_rows(n, ct):
    tb = fw.fw_host_pipeline_bounds(n, ct, 8)
    tiles = -(-n // 128)
    if not tb:
        assert ct == -1 and tiles < 32 or ct > 0 and tiles < 2 * ct
        return
    assert tb[0] == 0 and tb[-1] == tiles and len(tb) >= 3
    assert all(a < b for a, b in zip(tb, tb[1:]))
    sizes = np.diff(tb)
    if ct > 0:
        assert (sizes[:-1] == ct).all() and sizes[-1] <= ct
    elif tiles < 64:
        assert tb == [0, tiles // 2, tiles]
    else:
        assert sizes[0] == sizes[1] == 8
        assert all(b == 2 * a for a, b in zip(sizes[1:-2], sizes[2:-1]))
        assert sizes[-1] >= sizes[-2]


def test_bounds_auto_c4_and_errors():
    assert fw.fw_host_pipeline_bounds(16384, -1, 8) == [0, 8, 16, 32, 64, 128]
    assert fw.fw_host_pipeline_bounds(16384, -1, 16) == [0, 16, 32, 64, 128]
    assert fw.fw_host_pipeline_bounds(16384, 0, 8) == []
    assert fw.fw_host_pipeline_bounds(4096, -1, 8) == [0, 16, 32]  # 32..63 tile-rows: two halves
    assert fw.fw_host_pipeline_bounds(3968, -1, 8) == []          # < 32 tile-rows: not pipelined
    with pytest.raises(fw.FwError):
        fw.fw_host_pipeline_bounds(0, -1, 8)
    with pytest.raises(fw.FwError):
        fw.fw_host_pipeline_bounds(100, -2, 8)


def scaled_bounds(n_blocks, n_lib):
    """The library's auto geometry for a matrix of n_lib rows, mapped onto n_blocks blocks."""
    tb = fw.fw_host_pipeline_bounds(n_lib, -1, 8)
    tiles = tb[-1]
    return sorted(set(int(round(t * n_blocks / tiles)) for t in tb))


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("kind", ["complete_int", "er_int", "ring"])
def test_schedule_gives_the_oracle_distances(seed, kind):
    BS, nb = 4, 16                               # 16 blocks of 4 vertices: the C4 geometry / 8
    n = BS * nb
    if kind == "ring":
        W = gen.ring_with_chords(n, seed, 20, dtype=np.int32)
    elif kind == "er_int":
        W = gen.generate("er_int", n, 70 + seed, p=0.08, lo=1, hi=50)
    else:
        W = gen.generate("complete_int", n, 80 + seed).astype(np.int32)
    Dref = oracle.fw(W, None)[0].astype(np.int64)
    Dref[Dref >= gen.INF_I32] = INF
    for tb in (scaled_bounds(nb, 16384), [0, 1, 2, 4, 8, 16], [0, 5, 11, 16], [0, 8, 16]):
        D = run_pipeline(W, BS, tb)
        np.testing.assert_array_equal(D, Dref, err_msg=f"bounds {tb}")


def test_schedule_precondition_matters():
    """Reading pivot strips that have not completed their round (the last chunk skips its own
    pivot rounds) loses paths on a ring, whose shortest paths climb through every block: the
    model is sensitive to the precondition it certifies."""
    BS, nb = 4, 16
    n = BS * nb
    W = gen.ring(n, 1, dtype=np.int32)           # i -> i+1: paths pass through all later blocks
    Dref = oracle.fw(W, None)[0].astype(np.int64)
    D = run_pipeline(W, BS, [0, 4, 8, 16], violate=True)
    assert not np.array_equal(D, Dref)
    np.testing.assert_array_equal(run_pipeline(W, BS, [0, 4, 8, 16]), Dref)


@pytest.mark.parametrize("seed", range(3))
@pytest.mark.parametrize("kind", ["complete_int", "er_int", "ring"])
def test_pair_schedule_gives_the_oracle_distances(seed, kind):
    """Pairs of rounds in the model: the device schedule (one chunk, all rows)
    and the pipeline's (own pairs on wide chunks, plain pairs with partner-block batches) give
    the oracle's distances bit for bit."""
    BS, nb = 4, 16
    n = BS * nb
    if kind == "ring":
        W = gen.ring_with_chords(n, seed, 20, dtype=np.int32)
    elif kind == "er_int":
        W = gen.generate("er_int", n, 70 + seed, p=0.08, lo=1, hi=50)
    else:
        W = gen.generate("complete_int", n, 80 + seed).astype(np.int32)
    Dref = oracle.fw(W, None)[0].astype(np.int64)
    Dref[Dref >= gen.INF_I32] = INF
    for tb, min_rows in (([0, 16], 1), ([0, 2, 4, 8, 16], 4), ([0, 2, 4, 8, 16], 1), ([0, 8, 16], 1),
                         (scaled_bounds(nb, 16384), 4), ([0, 6, 10, 16], 4)):
        D = run_pipeline_pairs(W, BS, tb, min_rows)
        np.testing.assert_array_equal(D, Dref, err_msg=f"bounds {tb}")


def test_pair_schedule_needs_even_chunk_bounds():
    """A fused pair whose two pivot blocks lie in different chunks reads a pivot strip that has
    not completed the pair's second round: with odd chunk boundaries and the even-boundary
    condition dropped, paths are lost on a ring — the condition pipe_solve enforces."""
    BS, nb = 4, 16
    n = BS * nb
    W = gen.ring_with_chords(n, 0, 20, dtype=np.int32)
    Dref = oracle.fw(W, None)[0].astype(np.int64)
    tb = [0, 1, 2, 4, 8, 16]
    assert not np.array_equal(run_pipeline_pairs(W, BS, tb, 4, force=True), Dref)
    np.testing.assert_array_equal(run_pipeline_pairs(W, BS, tb, 4), Dref)


@pytest.mark.parametrize("seed", range(6))
def test_random_geometries(seed):
    """Random even chunk boundaries (and random odd ones, where plain pairs are switched off)
    and random pair thresholds: both schedules give the oracle's distances on random graphs."""
    rng = np.random.default_rng(300 + seed)
    BS, nb = 4, 16
    n = BS * nb
    W = gen.generate("er_int", n, 400 + seed, p=float(rng.choice([0.03, 0.08, 0.3])), lo=1, hi=40)
    Dref = oracle.fw(W, None)[0].astype(np.int64)
    Dref[Dref >= gen.INF_I32] = INF
    for _ in range(4):
        k = int(rng.integers(1, 5))
        even = bool(rng.integers(0, 2))
        pool = np.arange(2, nb, 2) if even else np.arange(1, nb)
        cuts = sorted(set(int(x) for x in rng.choice(pool, size=min(k, len(pool)), replace=False)))
        tb = [0] + cuts + [nb]
        np.testing.assert_array_equal(run_pipeline(W, BS, tb), Dref, err_msg=f"single {tb}")
        np.testing.assert_array_equal(run_pipeline_pairs(W, BS, tb, int(rng.integers(1, 9))), Dref,
                                      err_msg=f"pairs {tb}")

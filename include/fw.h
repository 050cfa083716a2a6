/*
 * fw.h — C ABI of the B200-native blocked Floyd–Warshall APSP library (libfwb200.so).
 *
 * Method: Rucci, De Giusti, Naiouf, "Blocked All-Pairs Shortest Paths Algorithm on
 * Intel Xeon Phi KNL Processor: A Case Study" (arxiv 1811.01201). Citations:
 *   P:n  = /root/reference/PAPER.md line n        S:n = SPEC.md line n
 *   BJ   = /root/repo/BASELINE.json (north_star)  R# = DESIGN.md "Readings of the paper"
 *
 * The operation (§3): given an n x n distance matrix D initialised with the
 * edge weights, for k = 0..n-1 relax D[i][j] = min(D[i][j], D[i][k] + D[k][j]); a path
 * matrix P is produced "when the reconstruction of the shortest path is required"
 * (P:78). The library computes it with the blocked algorithm of §4.1:
 * R = n_pad/BS rounds, each with phase 1 (diagonal block), phase 2 (pivot row
 * and column strips) and phase 3 (all remaining blocks).
 *
 * Conventions (DESIGN.md readings):
 *   R1  P is returned as a NEXT-HOP matrix by default (BJ:5 "next-hop");
 *       FW_PATH_LAST_K returns the paper's "most recently added intermediate node" form.
 *   R2  Relaxation is strict '<' (ties keep the old value).
 *   R3  No-edge sentinel: FP32 +INFINITY; INT32 FW_INF_I32 = 0x3FFFFFFF (INT32_MAX/2, BJ
 *       configs[2]). Unreachable outputs are exactly the sentinel, with next = -1.
 *   R4  The diagonal is forced to 0.
 *   R11 n is padded internally to a multiple of 128 with isolated vertices.
 *
 * Layout: every matrix is row-major and contiguous (leading dimension = n for host
 * buffers, `ld` elements for device buffers), element (i,j) at [i*ld + j].
 *
 * Errors: every function returns FW_OK (0) or a positive fw_status. fw_last_error()
 * returns a thread-local, human-readable message for the last non-OK return.
 *  - FW_EINVAL / FW_ERANGE are detected BEFORE any output is written: dist and next
 *    are left untouched.
 *  - After FW_ECUDA / FW_ENCCL the outputs are unspecified; call fw_free().
 *  - Calling fw_solve* before fw_init returns FW_ESTATE.
 * Ownership: the caller owns every buffer it passes; the library keeps no pointer to
 * them after a call returns. Device workspaces and streams live in the context created
 * by fw_init and are released by fw_free. Calls are serialised per process.
 */
#ifndef FW_B200_H
#define FW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FW_INF_I32 0x3FFFFFFF /* INT32 no-edge / unreachable sentinel (R3) */

enum fw_status {
  FW_OK = 0,
  FW_EINVAL = 1, /* bad argument or out-of-domain weight (negative, NaN, > FW_INF_I32) */
  FW_ENOMEM = 2, /* device or pinned-host allocation failed                          */
  FW_ECUDA = 3,  /* a CUDA runtime call or kernel failed                              */
  FW_ENCCL = 4,  /* NCCL (multi-GPU transport) unavailable or failed                    */
  FW_ESTATE = 5, /* fw_init not called, or called twice                               */
  FW_ERANGE = 6  /* INT32: (n-1) * max finite weight >= FW_INF_I32 (sums could hit INF) */
};

/* fw_init flags */
enum fw_flags {
  FW_PATH_NEXT_HOP = 0u,  /* P = next hop (default, R1)                          */
  FW_PATH_LAST_K = 1u,    /* P = last intermediate vertex k, -1 = direct edge */
  FW_TIMING = 2u          /* record per-phase CUDA-event times into fw_stats      */
};

/* Statistics of the last successful solve (fw_last_stats). Times in milliseconds. */
typedef struct fw_stats {
  int64_t n;            /* user n                                              */
  int64_t n_pad;        /* padded n (multiple of 128)                          */
  int32_t block;        /* BS used                                             */
  int32_t rounds;       /* rounds executed (rounds lying wholly in padding are skipped) */
  int32_t is_int;       /* 1 = INT32 solve                                     */
  int32_t path_mode;    /* -1 = no P, 0 = next hop, 1 = last k                 */
  int32_t p_method;     /* 0 = no P; 1 = round tags + post-pass (real-valued data);
                           2 = exact arg-min keys (integer-valued data)           */
  double solve_ms;      /* device-resident solve (init .. post-pass), CUDA events */
  double phase1_ms;     /* FW_TIMING only: sum over rounds                     */
  double phase2_ms;
  double phase3_ms;
  double post_ms;       /* P resolution post-pass                              */
  double h2d_ms;        /* host entry points only                              */
  double d2h_ms;
  int64_t phase3_launches; /* bulk phase-3 launches: one per round, or one per pair of rounds
                              when two rounds share a 256-deep pass       */
  double phase3_relaxations; /* relaxations issued by phase-3 launches (algorithmic) */
  int64_t kernel_launches; /* kernels this library launched for the solve (incl. validation) */
  int32_t compute_f32;  /* 1 = relaxations ran in FP32: FP32 data, or INT32 data whose stored
                           values are integers < 2^24 (exact in FP32)     */
  int32_t host_chunks;  /* host entry points: row chunks whose H2D / D2H overlapped the solve
                           (DESIGN.md §4.8); 0 = copies not overlapped. With a pipeline,
                           h2d_ms / d2h_ms are the EXPOSED parts (until the first chunk
                           landed / after the last chunk computed) and solve_ms the whole call */
  int64_t broadcasts;   /* ncclBroadcast calls this rank issued (pivot strips + the TAG-mode
                           post-pass gather); 0 without a communicator                    */
  double bcast_bytes;   /* bytes those broadcasts moved (per rank, as root or receiver)   */
  int32_t persistent;   /* 1 = the rounds ran as ONE persistent launch (work items ordered by
                           round, per-tile readiness counters): phase3_ms is
                           that launch (all phases) and phase3_relaxations = n_pad^3; 2 = the
                           same over a communicator with the pivot-row tiles published through
                           an NVLS multicast object (one multimem store reaches every rank)  */
} fw_stats;

/* Create the process-wide context. ngpus_max: the most devices one fw_solve may use,
 * 0 = all visible devices; the single-GPU entry points run on the calling thread's current
 * device. flags: FW_PATH_* | FW_TIMING. Returns FW_ESTATE if already initialised.
 * Schedule switches read here from the environment (tuning / A-B only; results are the same,
 * DESIGN.md §4.6-4.9): FW_LOOKAHEAD=0, FW_PAIRS=0 (one round per phase-3 pass),
 * FW_PAIR_ORDER=0, FW_PDL=0 (no programmatic dependent launch), FW_PIPE_FIRST=k,
 * FW_PIPE_PAIR_ROWS=k, FW_COPY_THREADS=k (host copy pool). */
int fw_init(int ngpus_max, unsigned flags);

/* Schedule switches of the live context (the same ones fw_init reads from the environment;
 * tuning, A/B comparisons and isolated per-phase timing — distances are identical, P valid):
 *   "lookahead"  0/1  phases 1-2 of round K+1 on the side stream under phase 3 of round K (§4.6)
 *   "pairs"      0/1  two rounds per phase-3 pass for keyed / distance-only solves (§4.9)
 *   "pdl"        0/1  programmatic dependent launch between consecutive phase-3 launches
 *   "pair_order" 0/1  the next pair's strips beside (1) or before (0) the bulk launch
 *   "pipe_pair_rows" k >= 1, "pipe_first" k in [1, 64]  host pipeline geometry (§4.8)
 *   "persistent" -1/0/1  the rounds of a one-GPU BS = 128 solve as ONE persistent launch whose
 *                        work items wait on per-tile round counters (§4.10): -1 auto (round-tag
 *                        solves), 0 off, 1 on (env FW_PERSISTENT)
 *   "persist_gap" k >= 0 persistent: phase-3 tiles between phase 1 and phase 2 of the next
 *                        round in the work order (-1 auto)
 *   "persist_relaxed" 0/1, "persist_quarters" -1/0/1/2  persistent: relaxed dependency polls;
 *                        critical-path tiles as 64 x 64 quarter items (one GPU; 1: every prio
 *                        and phase-2 tile, 2: the three tiles per round the pivot chain waits
 *                        for; -1 auto: 1 when n < 4096, else 2)
 *   "persist_p1_lone" -1/0/1  persistent, one GPU: one SM keeps a single CTA that runs every
 *                        phase-1 item (-1 auto = on, 0 off)
 *   "nvls"       -1/0/1  persistent over a communicator: publish the pivot-row tiles through an
 *                        NVLS multicast object when there are several ranks and every device
 *                        supports it (-1, default; set up collectively, any failure falls back
 *                        to the IPC peer rings), never (0), or try even with one rank (1: tests
 *                        the collective setup and its fallback on one GPU)
 *   "async"      0/1     fw_solve_device_* (one GPU) return as soon as the solve is enqueued on
 *                        the caller's stream: no validation kernel and no host round trip, so a
 *                        solve can be captured into a CUDA graph (after one warm-up solve of the
 *                        same size has allocated the workspaces). The caller guarantees the
 *                        domain (FP32: weights >= 0, no NaN; INT32: weights in [0, FW_INF_I32] and
 *                        (n-1) * max weight < FW_INF_I32) — outside it the results are undefined
 *                        instead of FW_EINVAL / FW_ERANGE. P comes from round tags (valid for every
 *                        such input; D is bitwise the keyed solve's for integer data). Device-side
 *                        failures (a dependency-wait timeout, non-converging next hops) are
 *                        returned by the next fw_last_stats, which also waits for the solve
 * FW_ESTATE before fw_init; FW_EINVAL for an unknown name or value. */
int fw_set_option(const char *name, int value);

/* Release every device buffer, stream and event of the context. Idempotent. */
int fw_free(void);

/* Host-memory solve, FP32.
 *   dist  in/out, n*n floats: W in (+inf = no edge, weights >= 0, no NaN), D out.
 *   next  out, n*n int32, or NULL for a distance-only solve. Next-hop mode: next[i][j] is
 *         the first vertex after i on a shortest i->j path, next[i][i] = i, -1 when j is
 *         unreachable. LAST_K mode: an intermediate k with D[i][j] = D[i][k] + D[k][j], or
 *         -1 for a direct edge, the diagonal, or an unreachable pair.
 *   n     number of vertices, 1 <= n <= 65536.
 *   block BS in {32, 64, 128}, or 0 = auto (128 for n >= 4096, else 64).
 *   ngpus 1 = the current device; G in [2, ngpus_max] = devices 0..G-1 of this process,
 *         block-row partitioned (BJ north_star; SURVEY §8 e): one host thread per device,
 *         an NCCL communicator over them (created on first use, kept until fw_free), the
 *         per-round pivot-strip broadcast, each device copying its own rows in and out;
 *         0 = ngpus_max. FW_EINVAL outside [0, ngpus_max]; FW_ESTATE while a
 *         fw_comm_init communicator (one process per GPU) is active; FW_ENCCL if NCCL
 *         cannot be loaded or initialised. A failing rank's message is prefixed with its
 *         rank and device.
 * Pinned (cudaHostAlloc/registered) buffers are copied directly; pageable buffers are
 * staged through an internal ring of pinned slices (fw_set_host_pipeline overlaps either
 * with the solve). */
int fw_solve(float *dist, int32_t *next, int64_t n, int block, int ngpus);

/* Host pipeline of the single-GPU host entry points. When block = 128 (any plan: keys, round tags, next == NULL; a speculative key run is
 * checked chunk by chunk before each chunk is copied out and falls back to the standard solve
 * from the device copy of the input; pageable host buffers are staged through a pinned ring
 * by a pool of copy threads, pinned ones are copied directly), the rows are split into chunks of `chunk_tiles` x 128 rows:
 * each chunk is copied in, validated and relaxed through the rounds whose pivots exist as soon
 * as it lands, and copied out as soon as it has finished, so the copies overlap the solve.
 * Results: D identical to the unpipelined solve (any order of rounds per row that reads
 * completed pivot strips gives the same distances: reading R16); P a valid next hop / last k
 * (ties may resolve differently). Error contract unchanged (validation completes before any
 * output is written). chunk_tiles: -1 = auto (chunks of 8, 8, 16, 32, .. tile-rows when n >= 8192,
 * two halves when 4096 <= n < 8192, else off),
 * 0 = off, k >= 1 = k tile-rows whenever the matrix has at least two chunks.
 * FW_ESTATE before fw_init; FW_EINVAL for chunk_tiles < -1. */
int fw_set_host_pipeline(int chunk_tiles);

/* Host-only (no GPU, no fw_init): the host pipeline's chunk boundaries for n, in tile-rows of
 * 128 (out[0] = 0 < out[1] < .. < out[C] = ceil(n/128)): chunk_tiles as fw_set_host_pipeline,
 * first_tiles the first chunk of the auto (-1) geometry (8 unless FW_PIPE_FIRST is set).
 * Returns the number of boundaries written (0 = that solve is not pipelined), or -FW_EINVAL
 * for bad arguments or max_out too small. */
int fw_host_pipeline_bounds(int64_t n, int chunk_tiles, int first_tiles, int32_t *out, int max_out);

/* Host-memory solve, INT32 (no-edge = FW_INF_I32; weights in [0, FW_INF_I32]). */
int fw_solve_i32(int32_t *dist, int32_t *next, int64_t n, int block, int ngpus);

/* Device-memory solve on the current device, enqueued on `stream` (a cudaStream_t; NULL =
 * legacy default stream). d_dist: n rows of `ld` >= n floats (in/out); d_next: n rows of
 * `ld` int32 or NULL. When n % 128 == 0 and ld == n the solve runs in place with no copy;
 * otherwise through an internal padded workspace. Returns after the solve completes
 * (the stream is synchronised: validation must finish before the rounds are issued). */
int fw_solve_device_f32(float *d_dist, int32_t *d_next, int64_t n, int64_t ld, int block,
                        void *stream);
int fw_solve_device_i32(int32_t *d_dist, int32_t *d_next, int64_t n, int64_t ld, int block,
                        void *stream);

/* ---- multi-GPU: one process per GPU (SURVEY §8 e; BJ north_star) ----------------------------
 * D and P are partitioned by contiguous block-rows: the n_pad/128 tile rows are split over
 * `world` ranks in ranges whose sizes differ by at most one. Each round the owner of the pivot
 * block-row runs phases 1-2 on it and broadcasts the pivot row strip (BS x n_pad elements,
 * ncclBroadcast over NVLink); every rank then updates its own rows (phase-2 column strip and
 * phase 3). This is the method's only exchange step; the look-ahead overlaps it with phase 3.
 *
 * fw_dist_partition: host-only (no GPU needed). Rows [row0, row0 + nrows) of the n x n matrix
 *   belong to `rank` (nrows = 0 when a rank gets only padding). Returns FW_EINVAL on bad args.
 * fw_dist_owner: rank owning (padded) global row `row`, or -1.
 * fw_comm_unique_id: fill out[128] with an NCCL unique id (call on one rank; the caller ships
 *   the bytes to the others, e.g. with torch.distributed). FW_ENCCL if NCCL cannot be loaded.
 * fw_comm_init: after fw_init, join the communicator of `world` ranks as `rank` on the current
 *   device. While a communicator is active only fw_dist_solve_* may solve; fw_comm_free
 *   returns the context to single-GPU use.
 * fw_dist_solve_device_f32/i32: collective; every rank calls it with the same n and block and
 *   its own rows: d_rows holds rows [row0, row0 + nrows) of the n x n input (row pitch ld >= n),
 *   overwritten with the same rows of D; d_next_rows (same shape, int32) receives P or is
 *   NULL on every rank. Errors are agreed on by all ranks (validation is all-reduced). */
int fw_dist_partition(int64_t n, int world, int rank, int64_t *row0, int64_t *nrows);
int fw_dist_owner(int64_t n, int world, int64_t row);
int fw_comm_unique_id(unsigned char *out);
int fw_comm_init(const unsigned char *id, int rank, int world);
int fw_comm_free(void);
int fw_dist_solve_device_f32(float *d_rows, int32_t *d_next_rows, int64_t n, int64_t ld, int block,
                             void *stream);
int fw_dist_solve_device_i32(int32_t *d_rows, int32_t *d_next_rows, int64_t n, int64_t ld,
                             int block, void *stream);

/* Loopback transport (testing the partitioned path on one GPU): every rank of a `world`-way
 * block-row partition is emulated in this process on `stream` — per-rank phase launches on its
 * own rows, the pivot-strip broadcast as a device copy into each rank's receive buffer, the
 * look-ahead tile split per rank. Same arguments and results as fw_solve_device_*; world in
 * [1, 64]. Not a performance path. */
int fw_dist_loopback_solve_device_f32(float *d_dist, int32_t *d_next, int64_t n, int64_t ld,
                                      int block, int world, void *stream);
int fw_dist_loopback_solve_device_i32(int32_t *d_dist, int32_t *d_next, int64_t n, int64_t ld,
                                      int block, int world, void *stream);

/* Path reconstruction (host-only, no GPU or fw_init needed): the vertices
 * of the shortest i -> j path encoded by the P matrix a solve returned (n x n int32, row-major,
 * host memory).
 *   mode FW_PATH_NEXT_HOP: i, next[i][j], next[next[i][j]][j], ..., j.
 *   mode FW_PATH_LAST_K:   the recursive expansion path(i,k) + path(k,j) of k = P[i][j], where
 *                          -1 is a direct edge (iterative: no recursion depth limit).
 * dist: the solve's D (FP32, or INT32 with dist_is_int32 = 1) for reachability (D[i][j] = INF:
 *   no path); required in LAST_K mode (-1 there also marks unreachable pairs), optional in
 *   next-hop mode (next = -1 marks them).
 * out: up to max_len vertices (i first, j last); out = NULL with max_len = 0 queries the length.
 * Returns the number of vertices (1 for i == j), 0 if j is unreachable from i, -FW_EINVAL for bad
 * arguments or a P that does not encode a path of at most n - 1 hops, -FW_ERANGE when the path
 * has more than max_len > 0 vertices (the first max_len are written). */
int64_t fw_path(const int32_t *P, const void *dist, int dist_is_int32, int64_t n, int64_t i, int64_t j,
                int mode, int32_t *out, int64_t max_len);

/* Host-only (no GPU, no fw_init): the work-item order of the persistent solve
 * for n vertices on a `world`-way block-row partition (world in [1, 8]); rank = -1: every rank's
 * items (the loopback grid), else that rank's subsequence (one GPU of a communicator); rank = -2
 * (world 1): the one-GPU kernel's own arithmetic decode of the order, run on the host; -3: the
 * same with the critical-path tiles as quarter items, -4: with only the three chain tiles per
 * round as quarter items ("persist_quarters" 1 / 2); gap = the phase-3 tiles placed between
 * P1(K+1) and the phase-2 items of round K+1. Each item is packed as
 * rank << 29 | type << 27 | K << 18 | I << 9 | J (type 1 = phase 1 on tile (K, K), 2 = tile (I, J)
 * relaxed through block K, 3 = a 64 x 64 quarter of it, the quarter in the rank bits). With out = NULL, max_out = 0 returns the count. Returns the number of
 * items, or -FW_EINVAL (bad arguments, max_out too small). For tests of the order's invariants. */
int64_t fw_persist_schedule(int64_t n, int world, int rank, int gap, uint32_t *out, int64_t max_out);

/* Message for the last non-OK return on this thread ("" if none). */
const char *fw_last_error(void);

/* Copy the statistics of the last successful solve. FW_ESTATE if none yet. */
int fw_last_stats(fw_stats *out);

/* Library version string, e.g. "fwb200 0.2 sm_100a". */
const char *fw_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FW_B200_H */

// fw_persist.cuh — the whole blocked Floyd–Warshall solve as ONE persistent launch (one GPU,
// BS = 128): SURVEY §8 row f1, the "persistent K3 polling per-block-row readiness" half.
//
// Method: arxiv 1811.01201 §4.1. Round K relaxes every tile (I, J) of
// 128 x 128 through block K: phase 1 on (K, K), phase 2 on row K and column K
// and phase 3 on the rest. The paper overlaps phases 2 and 3 of a round with OpenMP
// `nowait`; the stream-ordered driver (fw_api.cu) overlaps round K+1's pivot phases with
// round K's phase 3 through a second stream and a kernel boundary per round. Here there is no
// boundary at all: a grid of resident CTAs takes work items from one global counter, in a fixed
// order, and each item waits only for the tiles it reads, through per-tile round counters:
//
//   ver[I][J] = number of rounds tile (I, J) has completed (stored with release semantics after
//               the tile's stores; read with acquire before the tile is used as an operand).
//
// Items and what each waits for (a tile item of round K computes
//   D[I][J] <- min(D[I][J], D[I][K] (x) D[K][J])   (min-plus product through block K):
// the same product serves phase 2 (I == K: A is the closed diagonal block, B the tile itself;
// J == K: A the tile itself, B the diagonal block; reading R7) and phase 3):
//   P1(K)            ver[K][K] >= K                                 (phase 1, one CTA)
//   tile(K, I, J)    ver[I][J] >= K, ver[I][K] >= K+1 unless J == K, ver[K][J] >= K+1 unless I == K
// Item order (deadlock-free: every item waits only for items EARLIER in the order, which were
// taken by CTAs that are running — no co-residency assumption is needed):
//   P1(0), P2(0) tiles, then per round K a segment of T^2 items:
//     prio(K)  = phase-3 tiles of round K that round K+1's pivot phases read: tile (K+1, K+1)
//                first, then row K+1 (J != K), then column K+1 (I != K, K+1)      2T-3
//     P1(K+1)                                                                      1
//     rest(K)  = the other phase-3 tiles of round K, first part                   gap
//     P2(K+1)  = row K+1 (J != K+1) and column K+1 (I != K+1) of round K+1         2T-2
//     rest(K), second part                                                         (T-2)^2 - gap
//   (the last segment: the (T-1)^2 phase-3 tiles of round T-1, then no-ops).
// So round K+1's pivot path (P1, then P2) runs while round K's phase 3 drains — the cross-round
// look-ahead without a second stream — and round K+1's phase-3 tiles start tile by tile as soon
// as their operands are ready, not when the whole of round K has ended.
//
// Correctness with overlapping rounds (reading R16 of DESIGN.md): a tile may be read as an
// operand while its owner item rewrites it for a LATER round. Every stored value is the length of
// a real path and values only decrease (each 4-byte element is read either before or after its
// store), so a more-relaxed operand can only lower the result towards the true distance, never
// below it; keys and round tags stay valid by the triangle argument on the final D (R9). D is
// therefore bitwise the standard schedule's for integer data.
//
// Every operand read goes through L2 (cp.async.cg, ld.global.cg): tiles are written by other SMs
// and this SM's L1 may hold stale lines of them.
#pragma once
#include "fw_kernels.cuh"

namespace fwb {

constexpr int kMaxRanks = 8;   // ranks of one persistent grid (loopback) / of a team

// One rank's rows of a block-row partition (world = 1: all rows). Local row i of D / P is global
// row row0 + i; ver holds the round counters of the rank's tiles (tile-rows [t0, t1) x T);
// ring is the rank's pivot-row history: global rows of block K at ring + K*128*ldr, written by
// the owner of block K when those tiles are final for round K (the fused publish), with pub[K][J]
// = K + 1 once tile (K, J) is there. The owner reads its own pivot rows in place instead.
struct RankView {
  void *D;
  int32_t *P;
  int *ver;
  int *pub;
  void *ring;
  void *ring_mc;          // multicast address of the rings (NVLS), or null: per-peer stores
  int *pub_mc;
  int64_t row0;
  int t0, t1;
};

struct PersistArgs {
  int64_t ld;              // D / P pitch (elements)
  int64_t ldr;             // ring pitch (n_pad)
  int T;                   // tiles per dimension = rounds (BS = 128)
  int gap;                 // rest(K) tiles between P1(K+1) and P2(K+1)
  int world;               // ranks in rk[]
  const unsigned *items;   // packed item table (multi-rank), or null: the one-rank order, decoded
  unsigned long long *next;   // work counter (zeroed)
  int *maxkey;             // KEY: largest stored key (speculative key runs)
  int *flags;              // bit 5: a dependency wait timed out (the host fails the solve)
  long long total;         // number of items
  unsigned long long timeout_ns;
  int sync_relaxed;        // dependency polls with relaxed loads (A/B option; see the kernel)
  int p1_blocked;          // PLAIN / TAG phase 1 as the blocked closure (phase1_blocked_body)
  int quarters;            // one GPU: critical-path tiles as four 64 x 64 items (persist_decode)
  int *qcnt;               // per-tile count of finished quarters (zeroed)
  int stage_old;           // 128 x 128 tiles: the old tile staged in shared memory during the last
                           // chunk (tile_mainloop / tile_epilogue), 0: read from L2 in the epilogue
  int p1_lone;             // one GPU: the grid leaves one SM with a single CTA, which runs every
                           // P1 item alone on its SM (the others skip them); 0: off
  int *smcnt;              // p1_lone: per-SM count of resident CTAs, then the start barrier count
  int nsm;                 // SMs of the device
  unsigned long long *trace;   // per item {taken, operands ready, done} (%globaltimer ns) and
                               // (smid << 32 | blockIdx.x), or null (env FW_PERSIST_TRACE)
  RankView rk[kMaxRanks];
};

enum ItemType { IT_NONE = 0, IT_P1 = 1, IT_TILE = 2, IT_QTILE = 3 };
struct Item {
  int type, K, I, J, r;    // r: the rank whose rows hold tile (I, J); IT_QTILE: the quarter (0..3)
};
// packed item (host-built tables): rank 3 | type 2 | K 9 | I 9 | J 9 bits
__host__ __device__ __forceinline__ unsigned pack_item(int r, int type, int K, int I, int J) {
  return ((unsigned)r << 29) | ((unsigned)type << 27) | ((unsigned)K << 18) | ((unsigned)I << 9) | (unsigned)J;
}
__device__ __forceinline__ Item unpack_item(unsigned u) {
  return Item{(int)((u >> 27) & 3), (int)((u >> 18) & 511), (int)((u >> 9) & 511), (int)(u & 511), (int)(u >> 29)};
}

// Item `it` of the fixed order above (one GPU). With quarters (a.quarters = 1) every tile on
// the per-round critical path — round K+1's phase-2 tiles and the round-K tiles its phase 1 and
// phase 2 read (prio) — is split into four 64 x 64 items (quarter q: rows 64*(q>>1), columns
// 64*(q&1) of the tile, all 128 k), taken back to back: the chain P2(K) -> prio(K) -> P1(K+1)
// -> P2(K+1) then advances in quarter-tile steps, which at small n (C2) is the round's critical
// path. A tile's round counter advances when its fourth quarter is done.
// The rest(K) tiles (I, J not in {K, N = K+1}) in the order the items take them: first the tiles of
// row and column M = K+2 ((M, M) first) — their round-K values are what round N's prio tiles
// (tile (M, M), row M, column M), and through them P1(M), wait for — then the others row-major.
// (In plain row-major order the round-K version of (M, M) was an arbitrary rest tile, often in the
// second part, after P2(N): the per-round pivot chain waited for it, tools/persist_trace.py.)
__host__ __device__ __forceinline__ void persist_rest_ij(int q, int K, int T, int *I, int *J) {
  const int N = K + 1, M = K + 2, m = T - 2;
  if (M >= T) {
    *I = skip2(q / m, K, N);
    *J = skip2(q % m, K, N);
    return;
  }
  const int s = M - 2;                            // M's index among the rows / columns kept
  int ii, jj;
  if (q == 0) {
    ii = s, jj = s;
  } else if (q < m) {                             // row M
    ii = s;
    jj = q - 1 + (q - 1 >= s);
  } else if (q < 2 * m - 1) {                     // column M
    const int t = q - m;
    ii = t + (t >= s);
    jj = s;
  } else {
    const int t = q - (2 * m - 1);
    ii = t / (m - 1);
    jj = t % (m - 1);
    ii += ii >= s;
    jj += jj >= s;
  }
  *I = skip2(ii, K, N);
  *J = skip2(jj, K, N);
}

// quarters == 2 ("critical" quarters): only the three tiles per round that the pivot chain itself
// waits for are split — the round-K tile (N, N) that P1(N) reads (first in prio(K), N = K+1) and
// round N's phase-2 tiles (N, N+1), (N+1, N) that the next prio tile reads (first in P2(N)) — so
// the chain P1 -> P2 -> prio -> P1 advances in quarter steps while every other tile stays whole
// (the full quartering of prio / P2 costs more item overhead than it saves at T >= 32).
__host__ __device__ __forceinline__ long long persist_total_crit(int T) {
  if (T < 2) return 1;
  const long long m = T - 2, segA = 4LL * T + 5 + m * m, segB = 4LL * T - 1 + m * m;
  return 1 + (2LL * T + 4) + m * segA + segB + (long long)(T - 1) * (T - 1);
}
__host__ __device__ __forceinline__ Item persist_decode_crit(const PersistArgs &a, long long it) {
  const int T = a.T;
  const Item none{IT_NONE, 0, 0, 0, 0};
  if (it == 0) return Item{IT_P1, 0, 0, 0, 0};
  if (T < 2) return none;
  const long long pre = 1 + 2LL * T + 4;       // P1(0), P2(0): (0,1) x4, (1,0) x4, the rest whole
  if (it < pre) {
    const int q = (int)(it - 1);
    if (q < 4) return Item{IT_QTILE, 0, 0, 1, q};
    if (q < 8) return Item{IT_QTILE, 0, 1, 0, q - 4};
    const int t = q - 8;
    return t < T - 2 ? Item{IT_TILE, 0, 0, t + 2, 0} : Item{IT_TILE, 0, t - (T - 2) + 2, 0, 0};
  }
  const int m = T - 2;
  const long long segA = 4LL * T + 5 + (long long)m * m, segB = 4LL * T - 1 + (long long)m * m;
  long long r = it - pre;
  int K;
  long long ql;
  if (r < (long long)m * segA) {
    K = (int)(r / segA);
    ql = r - (long long)K * segA;
  } else if ((r -= (long long)m * segA) < segB) {
    K = T - 2;
    ql = r;
  } else {
    K = T - 1;
    ql = r - segB;
  }
  int q = (int)ql;
  if (K == T - 1) {                               // last round: its phase-3 tiles, then no-ops
    const int m1 = T - 1;
    if (q >= m1 * m1) return none;
    return Item{IT_TILE, K, skip2(q / m1, K, -1), skip2(q % m1, K, -1), 0};
  }
  const int N = K + 1;
  if (q < 4) return Item{IT_QTILE, K, N, N, q};  // prio: (N, N) in quarters, then row N, column N
  if (q < 2 * T) {
    const int t = q - 4;
    return t < T - 2 ? Item{IT_TILE, K, N, skip2(t, K, N), 0} : Item{IT_TILE, K, skip2(t - (T - 2), K, N), N, 0};
  }
  q -= 2 * T;
  if (q == 0) return Item{IT_P1, N, N, N, 0};
  q -= 1;
  const int rest = m * m, gap = a.gap < rest ? a.gap : rest;
  int ri, rj;
  if (q < gap) {
    persist_rest_ij(q, K, T, &ri, &rj);
    return Item{IT_TILE, K, ri, rj, 0};
  }
  q -= gap;
  if (N + 1 < T) {                                // P2(N): (N, N+1), (N+1, N) in quarters first
    if (q < 4) return Item{IT_QTILE, N, N, N + 1, q};
    if (q < 8) return Item{IT_QTILE, N, N + 1, N, q - 4};
    if (q < 2 * T + 4) {
      const int t = q - 8;
      return t < T - 2 ? Item{IT_TILE, N, N, skip2(t, N, N + 1), 0} : Item{IT_TILE, N, skip2(t - (T - 2), N, N + 1), N, 0};
    }
    q -= 2 * T + 4;
  } else {                                        // the last P2: whole tiles
    if (q < 2 * T - 2) {
      return q < T - 1 ? Item{IT_TILE, N, N, skip2(q, N, -1), 0} : Item{IT_TILE, N, skip2(q - (T - 1), N, -1), N, 0};
    }
    q -= 2 * T - 2;
  }
  q += gap;
  persist_rest_ij(q, K, T, &ri, &rj);
  return Item{IT_TILE, K, ri, rj, 0};
}

__host__ __device__ __forceinline__ Item persist_decode(const PersistArgs &a, long long it) {
  if (a.quarters == 2) return persist_decode_crit(a, it);
  const int T = a.T, Q = a.quarters ? 4 : 1, TQ = a.quarters ? IT_QTILE : IT_TILE;
  Item w{IT_NONE, 0, 0, 0, 0};
  if (it == 0) return Item{IT_P1, 0, 0, 0, 0};
  const long long pre = 1 + (long long)Q * 2 * (T - 1);   // P1(0) + the phase-2 tiles of round 0
  if (it < pre) {                                 // P2(0): row 0 (J = 1..T-1), column 0 (I = 1..T-1)
    const int q = (int)(it - 1), t = q / Q, qq = q % Q;
    return t < T - 1 ? Item{TQ, 0, 0, t + 1, qq} : Item{TQ, 0, t - (T - 1) + 1, 0, qq};
  }
  // (T^2 + 12 T) T + 8 T < 2^31 for T <= 512 (n <= 65536): 32-bit division
  const int seg = T * T + (Q - 1) * (4 * T - 5), r = (int)(it - pre);
  const int K = r / seg;
  int q = r - K * seg;
  if (K >= T) return w;
  if (K == T - 1) {                               // last round: its phase-3 tiles, then no-ops
    const int m = T - 1;
    if (q >= m * m) return w;
    return Item{IT_TILE, K, skip2(q / m, K, -1), skip2(q % m, K, -1), 0};
  }
  const int N = K + 1;
  if (q < Q * (2 * T - 3)) {                      // prio: row K+1 ((K+1, K+1) first), column K+1
    const int t = q / Q, qq = q % Q;
    if (t < T - 1) return Item{TQ, K, N, t == 0 ? N : skip2(t - 1, K, N), qq};
    return Item{TQ, K, skip2(t - (T - 1), K, N), N, qq};
  }
  q -= Q * (2 * T - 3);
  if (q == 0) return Item{IT_P1, N, N, N, 0};
  q -= 1;
  const int m = T - 2, rest = m * m;
  const int gap = a.gap < rest ? a.gap : rest;
  int ri, rj;
  if (q < gap) {
    persist_rest_ij(q, K, T, &ri, &rj);
    return Item{IT_TILE, K, ri, rj, 0};
  }
  q -= gap;
  if (q < Q * 2 * (T - 1)) {                      // P2(K+1): row K+1, then column K+1
    const int t = q / Q, qq = q % Q;
    return t < T - 1 ? Item{TQ, N, N, skip2(t, N, -1), qq} : Item{TQ, N, skip2(t - (T - 1), N, -1), N, qq};
  }
  q -= Q * 2 * (T - 1);
  q += gap;
  persist_rest_ij(q, K, T, &ri, &rj);
  return Item{IT_TILE, K, ri, rj, 0};
}

__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Spin (one thread) until *p >= v; bounded: after timeout_ns set bit 5 of *flags and give up.
__device__ __forceinline__ void wait_ge(const PersistArgs &a, const int *p, int v, unsigned long long t0) {
  while (ld_acquire(p) < v) {
    if (globaltimer() - t0 > a.timeout_ns) {
      atomicOr(a.flags, 32);
      return;
    }
    __nanosleep(64);
  }
}

template <typename T, int MODE>
__device__ __forceinline__ void persist_phase1(const PersistArgs &a, const RankView &v, int K, unsigned char *smem) {
  T *D = static_cast<T *>(v.D);
  const int kb = K * 128, r0 = (int)(kb - v.row0);
  if constexpr (std::is_same<T, float>::value && is_key(MODE)) {
    if (a.p1_blocked)
      phase1_blocked_key_body<true>(D, v.P, a.ld, r0, kb, a.maxkey, *reinterpret_cast<P1BSmem<float> *>(smem));
    else
      phase1_key_f32_body<128, 8, 8, true>(D, v.P, a.ld, r0, kb, a.maxkey, *reinterpret_cast<P1Smem<float, 128> *>(smem));
  } else if constexpr (!is_key(MODE)) {
    if (a.p1_blocked)
      phase1_blocked_body<T, MODE, true>(D, v.P, a.ld, r0, kb, K, *reinterpret_cast<P1BSmem<T> *>(smem));
    else
      phase1_pair_body<T, 128, MODE, 8, 8, true>(D, v.P, a.ld, r0, kb, K, *reinterpret_cast<P1Smem<T, 128> *>(smem));
  } else {
    phase1_body<T, 128, MODE, kP1Side, true>(D, v.P, a.ld, r0, kb, K, a.maxkey,
                                             *reinterpret_cast<P1Smem<T, 128> *>(smem));
  }
}

// The fused publish: tile (K, J) of the owner's rows is final for round K (phase
// 1 / the phase-2 row strip) — copy it into every other rank's pivot-row ring and raise that
// rank's pub[K][J] (system-scope release: the rings of a team live on peer GPUs, written over
// NVLink). With a multicast object (NVLS) one multimem store reaches every ring at once.
template <typename T>
__device__ __forceinline__ void persist_publish(const PersistArgs &a, int self, int K, int J) {
  using V = typename Vec4<T>::V;
  const RankView &o = a.rk[self];
  const T *src = static_cast<const T *>(o.D) + (int64_t)(K * 128 - o.row0) * a.ld + J * 128;
  const int64_t dst_off = (int64_t)K * 128 * a.ldr + J * 128;
  if (o.ring_mc) {   // NVLS: one multimem store per vector, replicated into every rank's ring
    float *dst = reinterpret_cast<float *>(static_cast<T *>(o.ring_mc) + dst_off);
    for (int e = threadIdx.x; e < 128 * 32; e += kThreads) {
      const int row = e >> 5, c4 = (e & 31) * 4;
      const V x = __ldcg(reinterpret_cast<const V *>(src + (int64_t)row * a.ld + c4));
      asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(dst + (int64_t)row * a.ldr + c4),
                   "f"(__int_as_float(Num<T>::bits(x.x))), "f"(__int_as_float(Num<T>::bits(x.y))),
                   "f"(__int_as_float(Num<T>::bits(x.z))), "f"(__int_as_float(Num<T>::bits(x.w)))
                   : "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      int *f = o.pub_mc + (int64_t)K * a.T + J;
      asm volatile("multimem.st.release.sys.global.b32 [%0], %1;" ::"l"(f), "r"(K + 1) : "memory");
    }
    return;
  }
  for (int q = 0; q < a.world; ++q) {
    if (q == self) continue;
    T *dst = static_cast<T *>(a.rk[q].ring) + dst_off;
    for (int e = threadIdx.x; e < 128 * 32; e += kThreads) {   // 128 rows x 32 float4
      const int row = e >> 5, c4 = (e & 31) * 4;
      const V x = __ldcg(reinterpret_cast<const V *>(src + (int64_t)row * a.ld + c4));
      __stcg(reinterpret_cast<V *>(dst + (int64_t)row * a.ldr + c4), x);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int q = 0; q < a.world; ++q) {
      if (q == self) continue;
      int *f = a.rk[q].pub + (int64_t)K * a.T + J;
      asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(f), "r"(K + 1) : "memory");
    }
  }
}

__device__ __forceinline__ int ld_relaxed(const int *p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int owner_rank(const PersistArgs &a, int K) {
  int o = 0;
  for (int q = 1; q < a.world; ++q)
    if (K >= a.rk[q].t0) o = q;
  return o;
}

// the staged old tile: 128 x 128 elements from stage (nch % kStages) = 1 on, within the allocation
static_assert((128 / kBK) % kStages == 1 && 2 * TileShape<128, 128>::kStage >= 128 * 128,
              "old-tile staging layout");

template <typename T, int MODE>
__global__ void __launch_bounds__(kThreads, 2)
fw_persistent_kernel(const PersistArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // s_cur: the item being processed, decoded once by thread 0 (the decode's integer divisions
  // would otherwise cost every thread ~10% of a tile's instructions); s_next: the next item index,
  // taken from the counter while the current one runs (hides the atomic's round trip; still
  // deadlock-free: the earliest unfinished item is always running, since a CTA holding a later
  // index is busy with an earlier item). Dynamic assignment balances the CTAs: a round-robin
  // static assignment measured 6% slower at C5.
  __shared__ Item s_cur;
  __shared__ long long s_next;
  __shared__ TileSrc<T> s_src;   // the current tile's operand origins (tile_mainloop)
  __shared__ long long s_it;     // the current item's index (trace)
  __shared__ unsigned long long s_t0, s_t1, s_ta, s_tb, s_tc;
  using S = TileShape<128, 128>;
  const int tid = threadIdx.x;
  // Dedicated phase-1 CTA (a.p1_lone, one GPU): the grid is one CTA short of two per SM, so one
  // SM holds a single CTA; every CTA registers its SM, a start barrier waits for the whole grid,
  // and the CTA alone on its SM runs every P1 item in round order (the critical path of a small
  // solve: the P1 -> P2 -> prio -> P1 chain) without sharing its SM with a tile
  // product; the other CTAs skip the P1 items of the order. If no SM ended up with one CTA, the
  // P1 items are taken as usual. Deadlock-free: P1(K) waits only for earlier items, and the
  // items waiting for P1(K) wait for a CTA that runs nothing else.
  __shared__ int s_lone;    // -1: no dedicated CTA, 0: a normal CTA, 1: this is the P1 CTA
  if (a.p1_lone) {
    if (tid == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      atomicAdd(a.smcnt + smid, 1);
      __threadfence();
      atomicAdd(a.smcnt + a.nsm, 1);
      const unsigned long long t0 = globaltimer();
      while (ld_acquire(a.smcnt + a.nsm) < (int)gridDim.x) {
        if (globaltimer() - t0 > a.timeout_ns) {
          atomicOr(a.flags, 32);
          break;
        }
        __nanosleep(128);
      }
      int lone_sm = -1;
      for (int q = 0; q < a.nsm && lone_sm < 0; ++q)
        if (ld_acquire(a.smcnt + q) == 1) lone_sm = q;
      s_lone = lone_sm < 0 ? -1 : ((int)smid == lone_sm ? 1 : 0);
    }
    __syncthreads();
  } else if (tid == 0) {
    s_lone = -1;
  }
  // the dedicated CTA walks the P1 items K = 0, 1, ... instead of the counter (s_next = K)
  if (tid == 0) s_next = s_lone == 1 ? 0 : (long long)atomicAdd(a.next, 1ull);
  for (;;) {
    __syncthreads();   // the previous item is done with s_cur
    if (tid == 0) {
      const long long it = s_next;
      if (s_lone == 1) {                               // the dedicated P1 CTA
        s_cur = it < a.T ? Item{IT_P1, (int)it, (int)it, (int)it, 0} : Item{-1, 0, 0, 0, 0};
        s_next = it + 1;
        if (a.trace) s_it = a.total + it, s_t0 = globaltimer();   // its records follow the items
      } else if (it < a.total) {
        if (a.trace) s_it = it, s_t0 = globaltimer();
        s_next = (long long)atomicAdd(a.next, 1ull);
        Item w = a.items ? unpack_item(a.items[it]) : persist_decode(a, it);
        if (w.type == IT_P1 && s_lone == 0) w.type = IT_NONE;   // the dedicated CTA's
        s_cur = w;
        if (a.trace) s_ta = globaltimer();
        if (w.type == IT_QTILE) {   // one GPU: rows / columns 64 * (quarter bits) of tile (I, J)
          const RankView &v = a.rk[0];
          const T *Dv = static_cast<const T *>(v.D);
          const int qi = (w.r >> 1) * 64, qj = (w.r & 1) * 64;
          s_src.a = Dv + (int64_t)(w.I * 128 + qi) * a.ld + w.K * 128;
          s_src.lda = a.ld;
          s_src.b = Dv + (int64_t)w.K * 128 * a.ld + w.J * 128 + qj;
          s_src.ldb = a.ld;
          s_src.old = nullptr;
        }
        if (w.type == IT_TILE) {   // A = (I, K) of this rank's rows; B = (K, J) in place or the ring
          const RankView &v = a.rk[w.r];
          const bool own_b = w.K >= v.t0 && w.K < v.t1;
          const T *Dv = static_cast<const T *>(v.D);
          s_src.a = Dv + (int64_t)(w.I - v.t0) * 128 * a.ld + w.K * 128;
          s_src.lda = a.ld;
          s_src.b = own_b ? Dv + (int64_t)(w.K - v.t0) * 128 * a.ld + w.J * 128
                          : static_cast<const T *>(v.ring) + (int64_t)w.K * 128 * a.ldr + w.J * 128;
          s_src.ldb = own_b ? a.ld : a.ldr;
          s_src.old = a.stage_old ? Dv + (int64_t)(w.I - v.t0) * 128 * a.ld + w.J * 128 : nullptr;
          s_src.ldo = a.ld;
        }
      } else {
        s_cur = Item{-1, 0, 0, 0, 0};
      }
    }
    __syncthreads();
    if (a.trace && tid == 0) s_tb = globaltimer();
    const Item w = s_cur;
    if (w.type < 0) break;
    if (w.type == IT_NONE) continue;
    const RankView &v = a.rk[w.type == IT_QTILE ? 0 : w.r];
    T *D = static_cast<T *>(v.D);
    const int li = w.I - v.t0;                      // local tile-row of the item's tile
    if (w.type == IT_TILE) {
      // warm L2 with the tile for the epilogue's compare (read once per round from HBM; its
      // latency is otherwise the epilogue's top stall), as the stream-ordered kernel does.
      // Placed after the dependency polls or left out, C2 is the same (4.64 ms either way).
      for (int l = tid; l < 128 * 4; l += kThreads)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(D + (int64_t)(li * 128 + l / 4) * a.ld + w.J * 128 + (l % 4) * 32));
    }
    if (tid < 3) {   // the operands this item reads and its own tile at the required round: one
                     // thread per counter, so the three loads are in flight together
      const int64_t T_ = a.T;
      const int *p = nullptr;
      int need = 0;
      if (w.type == IT_P1) {
        if (tid == 0) p = v.ver + li * T_ + w.K, need = w.K;
      } else if (tid == 0) {
        p = v.ver + li * T_ + w.J, need = w.K;                      // own tile, round K-1 done
      } else if (tid == 1) {
        if (w.J != w.K) p = v.ver + li * T_ + w.K, need = w.K + 1;  // A = (I, K), this rank's rows
      } else if (w.I != w.K) {                                     // B = (K, J): in place on the
        const bool own = w.K >= v.t0 && w.K < v.t1;                // owner, else the ring
        p = own ? v.ver + (int64_t)(w.K - v.t0) * T_ + w.J : v.pub + w.K * T_ + w.J;
        need = w.K + 1;
      }
      if (p) {
        // acquire (LDG.STRONG + an L1 invalidate), or relaxed when every operand read of the
        // kernel bypasses L1 anyway (cp.async.cg / ld.global.cg: a_sync_relaxed, A/B option)
        int val = a.sync_relaxed ? ld_relaxed(p) : ld_acquire(p);
        if (val < need) {
          const unsigned long long t0 = globaltimer();
          while ((val = a.sync_relaxed ? ld_relaxed(p) : ld_acquire(p)) < need) {
            if (globaltimer() - t0 > a.timeout_ns) {
              atomicOr(a.flags, 32);
              break;
            }
            __nanosleep(64);
          }
        }
      }
    }
    if (a.trace && tid == 0) s_tc = globaltimer();
    __syncthreads();
    if (a.trace && tid == 0) s_t1 = globaltimer();
    if (w.type == IT_P1) {
      persist_phase1<T, MODE>(a, v, w.K, smem_raw);
    } else if (w.type == IT_QTILE) {
      using S64 = TileShape<64, 64>;
      T acc[S64::RM][4 * S64::H];
      tile_mainloop<T, 64, 64>(reinterpret_cast<T *>(smem_raw), &s_src, 128 / kBK, acc);
      const Item e = s_cur;
      int kmax = tile_epilogue<T, 64, 64, MODE, true>(D, a.rk[0].P, a.ld, e.I * 128 + (e.r >> 1) * 64,
                                                      e.J * 128 + (e.r & 1) * 64, 0, 0, 0, 0, e.K,
                                                      (e.K * 128) & ~kKeyMask, acc);
      if (is_key(MODE)) {
        kmax = __reduce_max_sync(0xffffffffu, kmax);
        if ((tid & 31) == 0 && kmax > 0) atomicMax(a.maxkey, kmax);
      }
    } else {
      T acc[S::RM][4 * S::H];
      tile_mainloop<T, 128, 128>(reinterpret_cast<T *>(smem_raw), &s_src, 128 / kBK, acc);
      // the item again from shared memory: nothing but the accumulators lives across the loop
      const Item e = s_cur;
      const RankView &ve = a.rk[e.r];
      const T *old_s = nullptr;
      if (s_src.old) {   // the staged old tile (stages 1-2 of the last chunk, 128 / kBK = 4 chunks)
        cp_async_wait<0>();
        __syncthreads();
        old_s = reinterpret_cast<const T *>(smem_raw) + ((128 / kBK) % kStages) * S::kStage;
      }
      int kmax = tile_epilogue<T, 128, 128, MODE, true>(static_cast<T *>(ve.D), ve.P, a.ld, (e.I - ve.t0) * 128,
                                                        e.J * 128, 0, 0, 0, 0, e.K, (e.K * 128) & ~kKeyMask, acc,
                                                        old_s);
      if (is_key(MODE)) {
        kmax = __reduce_max_sync(0xffffffffu, kmax);
        if ((tid & 31) == 0 && kmax > 0) atomicMax(a.maxkey, kmax);
      }
    }
    __syncthreads();   // every thread's stores of the tile precede the release below (bar.sync
                       // orders them before thread 0's release, which is cumulative)
    const Item e = s_cur;
    if (a.world > 1 && e.I == e.K) persist_publish<T>(a, e.r, e.K, e.J);   // a final pivot-row tile
    if (tid == 0) {
      const RankView &ve = a.rk[e.type == IT_QTILE ? 0 : e.r];
      int *vp = ve.ver + (int64_t)(e.I - ve.t0) * a.T + e.J;
      bool last = true;
      if (e.type == IT_QTILE) {   // the tile is done for round K when its fourth quarter is
        __threadfence();          // this quarter's stores before its count
        last = (atomicAdd(a.qcnt + (int64_t)e.I * a.T + e.J, 1) & 3) == 3;
      }
      if (last) asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(vp), "r"(e.K + 1) : "memory");
      if (a.trace) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        unsigned long long *rec = a.trace + 8 * s_it;
        rec[0] = s_t0;
        rec[1] = s_t1;
        rec[2] = globaltimer();
        rec[3] = ((unsigned long long)smid << 32) | blockIdx.x;
        rec[4] = s_ta;   // decoded (thread 0)
        rec[5] = s_tb;   // past the barrier after the decode
        rec[6] = s_tc;   // thread 0's dependency poll done
      }
    }
  }
}

}  // namespace fwb

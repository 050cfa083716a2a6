// fw_kernels.cuh — sm_100a kernels of the blocked Floyd–Warshall hot path.
//
// Method: arxiv 1811.01201 §4.1. Round K relaxes every pair through
// the BS intermediate vertices k in [kb, kb+BS), kb = K*BS, in three phases:
//   phase 1     diagonal block D_KK, self-dependent: sequential k-loop in smem
//   phase 2 pivot row strip D_KJ and column strip D_IK, each relaxed through
//                        the closed D_KK* as a min-plus product (reading R7)
//   phase 3     every other block D_IJ <- min(D_IJ, D_IK (x) D_KJ)
// In phases 2 and 3 the element (i,j) is relaxed through A(i,k) = D[i][kb+k] and
// B(k,j) = D[kb+k][j] (global coordinates), so one tile kernel serves all three launches.
//
// The loop body of the paper's FW_BLOCK ("one addition, one comparison") becomes
// the relaxation microkernel: FP32 uses FADD2 with a broadcast scalar a_ik against a pair
// (b_kj, b_k,j+1) — two relaxations per instruction — and FMNMX3 folding the candidates
// of two consecutive k into the accumulator (two mins per instruction): one issue slot
// per relaxation. INT32 uses VIADDMNMX (fused add+min, one per relaxation).
//
// P modes (reading R9):
//   PLAIN   distances only.
//   KEY_*   integer-valued data: every stored value is a key D' = D*256 + (column & 255).
//           A candidate a'_ik + b'_kj = (D_ik + D_kj)*256 + (k&255) + (j&255), so the
//           minimum over k is the minimum distance AND, among ties, the smallest k — the
//           arg-min comes for free with the same instruction count. The epilogue recovers
//           k, stores D' = sum - (k&255) and P[i][j] = k (the paper's last intermediate
//           vertex); a per-row pointer-jumping pass turns it into next hops.
//           Exact while every key sum stays below 2^24 (FP32) / 2^30 (INT32); the host
//           verifies the bound (statically, or from the max stored key after the solve).
//   TAG     real-valued data: the epilogue writes the round number K for every element
//           that strictly improved; a post-pass resolves tags into P.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include <type_traits>

namespace fwb {

constexpr int kThreads = 256;         // tile kernel: 256 threads
constexpr int kBK = 32;               // k-chunk staged per pipeline stage
constexpr int kStages = 3;            // cp.async pipeline depth (one barrier per chunk)
constexpr int kTerm = 0x40000000;     // terminal bit used by the next-hop pointer jumping
constexpr int kP1Side = 16;           // phase 1: kP1Side^2 threads, (BS/kP1Side)^2 elements each
// Key encoding: a stored key is D * kKeyMul + (column & kKeyMask); the low
// kKeyBits bits of a candidate sum carry k within a 256-aligned window of two 128-blocks, so a
// single pass may relax through up to 256 consecutive k (two rounds of BS = 128).
constexpr int kKeyBits = 8;
constexpr int kKeyMul = 1 << kKeyBits;
constexpr int kKeyMask = kKeyMul - 1;

enum Mode { MODE_PLAIN = 0, MODE_TAG = 1, MODE_KEY = 2 };
__host__ __device__ constexpr bool is_key(int m) { return m == MODE_KEY; }

template <typename T> struct Num;
template <> struct Num<float> {
  static constexpr bool kIsInt = false;
  static __device__ __forceinline__ float inf() { return __int_as_float(0x7f800000); }
  static __device__ __forceinline__ float acc_init() { return __int_as_float(0x7f800000); }
  static __device__ __forceinline__ bool bad(float v) { return !(v >= 0.0f); }  // NaN or < 0
  static __device__ __forceinline__ bool finite(float v) { return v < inf(); }
  static __device__ __forceinline__ int lowk(float v) { return (int)v & kKeyMask; }   // v < 2^24
  static __device__ __forceinline__ float from_int(int v) { return (float)v; }
  static __device__ __forceinline__ int bits(float v) { return __float_as_int(v); }
  static __device__ __forceinline__ float encode(float v, int col) {       // key D*256 + col'
    return finite(v) ? v * (float)kKeyMul + (float)(col & kKeyMask) : v;
  }
  static __device__ __forceinline__ float decode(float k) { return finite(k) ? floorf(k * (1.0f / kKeyMul)) : k; }
};
template <> struct Num<int32_t> {
  static constexpr bool kIsInt = true;
  static __device__ __forceinline__ int32_t inf() { return 0x3FFFFFFF; }
  static __device__ __forceinline__ int32_t acc_init() { return 0x7FFFFFFF; }
  static __device__ __forceinline__ bool bad(int32_t v) { return v < 0 || v > 0x3FFFFFFF; }
  static __device__ __forceinline__ bool finite(int32_t v) { return v < 0x3FFFFFFF; }
  static __device__ __forceinline__ int lowk(int32_t v) { return v & kKeyMask; }
  static __device__ __forceinline__ int32_t from_int(int v) { return v; }
  static __device__ __forceinline__ int bits(int32_t v) { return v; }
  static __device__ __forceinline__ int32_t encode(int32_t v, int col) {
    return finite(v) ? v * kKeyMul + (col & kKeyMask) : v;
  }
  static __device__ __forceinline__ int32_t decode(int32_t k) { return finite(k) ? (k >> kKeyBits) : k; }
};

template <typename T> struct Vec4;
template <> struct Vec4<float> { using V = float4; };
template <> struct Vec4<int32_t> { using V = int4; };

template <typename V> __device__ __forceinline__ auto vget(const V &v, int e) {
  return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
}
template <typename V, typename S> __device__ __forceinline__ void vset(V &v, int e, S x) {
  if (e == 0) v.x = x; else if (e == 1) v.y = x; else if (e == 2) v.z = x; else v.w = x;
}

// ---------------------------------------------------------------------------------
// cp.async helpers (LDGSTS): global -> shared without staging registers.
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------------
// Relaxation microkernels. x0..x3: accumulators of one row i and four consecutive
// columns j..j+3; a0, a1 = a_ik, a_i,k+1; b0, b1 = B[k][j..j+3], B[k+1][j..j+3].
// Folds the 8 candidates a_ik + b_kj (one IEEE round-to-nearest add each) into x by min.
// min is exact, so the fold order does not change the result (reading R8).
__device__ __forceinline__ void relax2k(float &x0, float &x1, float &x2, float &x3, float a0,
                                        float a1, const float4 &b0, const float4 &b1) {
  const float2 s0 = __fadd2_rn(make_float2(a0, a0), make_float2(b0.x, b0.y));  // FADD2, a0 broadcast
  const float2 s1 = __fadd2_rn(make_float2(a1, a1), make_float2(b1.x, b1.y));
  const float2 s2 = __fadd2_rn(make_float2(a0, a0), make_float2(b0.z, b0.w));
  const float2 s3 = __fadd2_rn(make_float2(a1, a1), make_float2(b1.z, b1.w));
  x0 = fminf(x0, fminf(s0.x, s1.x));                                            // FMNMX3
  x1 = fminf(x1, fminf(s0.y, s1.y));
  x2 = fminf(x2, fminf(s2.x, s3.x));
  x3 = fminf(x3, fminf(s2.y, s3.y));
}
__device__ __forceinline__ void relax2k(int &x0, int &x1, int &x2, int &x3, int a0, int a1,
                                        const int4 &b0, const int4 &b1) {
  x0 = __viaddmin_s32(a0, b0.x, x0);  // VIADDMNMX: min(a+b, x)
  x1 = __viaddmin_s32(a0, b0.y, x1);
  x2 = __viaddmin_s32(a0, b0.z, x2);
  x3 = __viaddmin_s32(a0, b0.w, x3);
  x0 = __viaddmin_s32(a1, b1.x, x0);
  x1 = __viaddmin_s32(a1, b1.y, x1);
  x2 = __viaddmin_s32(a1, b1.z, x2);
  x3 = __viaddmin_s32(a1, b1.w, x3);
}

// Thread layout of a TM x TN tile: TX threads across (each owns H groups of 4 consecutive
// columns, 4*TX apart), TY = 256/TX threads down (each owns RM rows, TY apart).
template <int TM, int TN>
struct TileShape {
  static constexpr int H = TN >= 128 ? 2 : 1;
  static constexpr int TX = TN / (4 * H);
  static constexpr int TY = kThreads / TX;
  static constexpr int RM = TM / TY;
  static constexpr int AS = kBK + 4;                  // padded A row: conflict-free LDS.128
  static constexpr int BSTR = TN;                     // B row stride
  static constexpr int kA = TM * AS;
  static constexpr int kB = kBK * BSTR;
  static constexpr int kStage = kA + kB;
  static constexpr int kBytes = kStages * kStage * 4;
  static constexpr int kMinBlocks = TM * TN > 128 * 128 ? 1 : (TM * TN == 128 * 128 ? 2 : 3);
  static_assert(TX * TY == kThreads && RM >= 1 && RM * TY == TM, "tile shape");
};

// Launch arguments of the tile kernel (passed by value).
struct TileArgs {
  int64_t ld;
  const void *B;                 // B(k, j) = B[k * ldb + j]: the pivot row strip (rows kb..kb+Kd)
  int64_t ldb;
  int kb, Kd;
  int rows_lim, cols_lim;        // local rows / columns of D (tiles beyond them exit)
  int row0[2], col0[2];          // tile grid origin (local row, global column), per blockIdx.z
  int mr_lo[2], mr_hi[2];        // excluded rows, per blockIdx.z
  int mc_lo[2], mc_hi[2];        // excluded columns, per blockIdx.z
  int xrow[2];                   // 1: blockIdx.x walks tile rows (column strip in a dual launch)
  int tag;                       // round number (TAG mode)
  // Column-strip batch (host pipeline, BS = 128): every CTA relaxes its tile
  // through the block of its own columns, k in [j0, j0 + 128): A = the tile itself, B = rows
  // j0.. of the matrix whose row 0 is at g.B (pitch ldb), tag = j0 / 128 (that block's round).
  int colstrip;                  // 2: through the PARTNER block of a 256-aligned pair (j0 ^ 128)
  int colstep;                   // tile-column stride of the grid (0 or 1: consecutive)
  // Ordered phase-3 launch (order = 1, 1-D grid, 128 x 128 tiles): blockIdx.x enumerates the
  // round's tiles with the look-ahead set first — A1 = tile-row rowN (next pivot block-row,
  // -1 if not local) except tile-column colK; A2 = tile-column colN except tile-rows rowK and
  // rowN; then B = every tile outside tile-rows {rowK, rowN} and tile-columns {colK, colN}.
  // The CTAs of A1 + A2 (the first nprio) count themselves into *done after their stores, so
  // the next round's pivot phases can start while B is still running.
  int order;
  int tiles_r, tiles_c;          // local tile-rows, tile-columns
  int rowK, rowN, colK, colN;    // local tile-row of pivot blocks K / K+1 (-1: not local); tile-columns
  int nprio;                     // |A1| + |A2|
  int *done;                     // per-round counter of finished look-ahead tiles
};

// k-th element of {0, .., n-1} \ {x, y} (x, y < 0 or distinct: not excluded twice)
__host__ __device__ __forceinline__ int skip2(int k, int x, int y) {
  const int lo = (x >= 0 && y >= 0) ? min(x, y) : max(x, y), hi = (x >= 0 && y >= 0) ? max(x, y) : -1;
  if (lo >= 0 && k >= lo) ++k;
  if (hi >= 0 && k >= hi) ++k;
  return k;
}

// ---------------------------------------------------------------------------------
// Min-plus tile kernel (phases 2 and 3). Tile origin (i0, j0) = (row0 + by*TM, col0 + bx*TN);
// blockIdx.z selects one of two strip descriptions (phase 2 launches both strips at once).
//   D[i][j] <- min(D[i][j], min_{k<Kd} D[i][kb+k] + B[k][j])
// with i a LOCAL row of this GPU's block-row partition (all rows on one GPU) and B the pivot
// row strip (rows kb..kb+Kd of the global matrix: in D on its owner, the broadcast buffer
// elsewhere), for the tile's (i,j), excluding rows in [mr_lo, mr_hi) and columns in [mc_lo, mc_hi)
// (strips owned by other phases). The k dimension is streamed in chunks of kBK
// through kStages shared-memory stages (cp.async 16 B): A row-major [i][k] (padded), B row-major
// [k][j]. In-place use (phase 2: the tile is its own A or B) is safe: a CTA reads all its
// A/B chunks before its epilogue writes, and no other CTA writes what it reads.
// Tile origin (local row, global column) and excluded rows / columns of one CTA of a tile
// launch; skip = the tile lies in an excluded strip or outside the local rows / columns.
struct TileSlot {
  int i0, j0, mr_lo, mr_hi, mc_lo, mc_hi;
  bool skip;
};

template <int TM, int TN, bool DUAL, bool STEP = true>
__device__ __forceinline__ TileSlot tile_slot(const TileArgs &g, int bxr, int byr, int bzr) {
  TileSlot t{};
  // select the strip description without dynamic indexing (keeps g out of local memory)
  const bool z = DUAL && bzr != 0;
  if (!DUAL && TM == 128 && TN == 128 && g.order) {   // ordered phase 3: the tile list above
    int q = bxr, by, bx;
    const int nA1 = g.rowN >= 0 ? g.tiles_c - 1 : 0;
    const int nA2 = g.tiles_r - (g.rowK >= 0) - (g.rowN >= 0);
    if (q < nA1) {
      by = g.rowN;
      bx = skip2(q, g.colK, -1);
    } else if ((q -= nA1) < nA2) {
      by = skip2(q, g.rowK, g.rowN);
      bx = g.colN;
    } else {
      q -= nA2;
      const int nc = g.tiles_c - 2;
      by = skip2(q / nc, g.rowK, g.rowN);
      bx = skip2(q % nc, g.colK, g.colN);
    }
    t.i0 = by * TM;
    t.j0 = bx * TN;
    t.skip = false;
    return t;
  }
  t.mr_lo = z ? g.mr_lo[1] : g.mr_lo[0];
  t.mr_hi = z ? g.mr_hi[1] : g.mr_hi[0];
  t.mc_lo = z ? g.mc_lo[1] : g.mc_lo[0];
  t.mc_hi = z ? g.mc_hi[1] : g.mc_hi[0];
  const int xrow = z ? g.xrow[1] : g.xrow[0];
  const int bx = xrow ? byr : bxr, by = xrow ? bxr : byr;   // xrow: blockIdx.y steps tile columns
  t.i0 = (z ? g.row0[1] : g.row0[0]) + by * TM;
  if constexpr (STEP) t.j0 = (z ? g.col0[1] : g.col0[0]) + bx * TN * (g.colstep > 1 ? g.colstep : 1);
  else t.j0 = (z ? g.col0[1] : g.col0[0]) + bx * TN;
  t.skip = (t.i0 >= t.mr_lo && t.i0 + TM <= t.mr_hi) || (t.j0 >= t.mc_lo && t.j0 + TN <= t.mc_hi) ||
           t.i0 >= g.rows_lim || t.j0 >= g.cols_lim;
  return t;
}

// blockIdx through inline asm: the epilogue recomputes its tile slot instead of keeping it
// live in registers across the main loop (the loop needs all 128).
__device__ __forceinline__ int ctaid(int dim) {
  int v;
  if (dim == 0) asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(v));
  else if (dim == 1) asm volatile("mov.u32 %0, %%ctaid.y;" : "=r"(v));
  else asm volatile("mov.u32 %0, %%ctaid.z;" : "=r"(v));
  return v;
}

// ---- the tile product of the persistent kernel (fw_persist.cuh) ---------------------------------
// Operand origins of one tile, in shared memory: A(i, k) = a[i*lda + k] (the tile's rows of the
// pivot column block), B(k, j) = b[k*ldb + j] (the pivot row block's columns of the tile).
template <typename T> struct TileSrc {
  const T *a;
  const T *b;
  int64_t lda, ldb;
  const T *old;      // or null: the tile itself (TM x TN at pitch ldo), staged into the free
  int64_t ldo;       // shared-memory stages during the last chunk for the epilogue's compare
};

// Main loop of one TM x TN tile: acc[r][c] = min over k < nch*kBK of A(i, k) + B(k, j) for the
// thread's rows i = ty + TY*r and columns j = 4*tx + 4*TX*h + e. The k dimension is streamed in
// chunks of kBK through kStages shared-memory stages (cp.async 16 B, .cg: through L2, never a
// stale L1 line): A row-major [i][k] (padded stride: conflict-free LDS.128), B row-major [k][j];
// one barrier per chunk. The cp.async source addresses are recomputed every chunk from `src`
// (shared memory) and a fresh %tid.x, so no address lives across the loop: with them live, the
// 128-register allocation spilled them and reloaded them after every chunk's barrier (the
// pattern that cost the stream kernel 6%). The same arithmetic as the stream
// kernel below (which writes it out to keep its spill-free allocation).
template <typename T, int TM, int TN>
__device__ __forceinline__ void tile_mainloop(T *smem, const TileSrc<T> *src, int nch,
                                              T (&acc)[TileShape<TM, TN>::RM][4 * TileShape<TM, TN>::H]) {
  using S = TileShape<TM, TN>;
  using V = typename Vec4<T>::V;
  constexpr int RM = S::RM, H = S::H, TX = S::TX, TY = S::TY;
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  // cp.async assignments: A chunk TM x kBK, B chunk kBK x TN, 16 B per copy.
  constexpr int A_PER = TM * (kBK / 4) / kThreads;
  constexpr int A_ROWS = kThreads / (kBK / 4);
  constexpr int B_PER = kBK * (TN / 4) / kThreads;
  constexpr int B_ROWS = kThreads / (TN / 4);
  static_assert(A_PER >= 1 && B_PER >= 1, "copy mapping");

  auto load_chunk = [&](int stage, int k0) {
    T *as = smem + stage * S::kStage;
    T *bs = as + S::kA;
    int tv;
    asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tv));
    const int ar = tv / (kBK / 4), ac = (tv % (kBK / 4)) * 4, br = tv / (TN / 4), bc = (tv % (TN / 4)) * 4;
    const int64_t lda = src->lda, ldb = src->ldb;
    const T *asrc = src->a + (int64_t)ar * lda + ac;
    const T *bsrc = src->b + (int64_t)br * ldb + bc;
#pragma unroll
    for (int t = 0; t < A_PER; ++t)
      cp_async16(as + (ar + t * A_ROWS) * S::AS + ac, asrc + k0 + (int64_t)t * A_ROWS * lda);
#pragma unroll
    for (int t = 0; t < B_PER; ++t)
      cp_async16(bs + (br + t * B_ROWS) * S::BSTR + bc, bsrc + (int64_t)(k0 + t * B_ROWS) * ldb);
    cp_async_commit();
  };

#pragma unroll
  for (int r = 0; r < RM; ++r)
#pragma unroll
    for (int c = 0; c < 4 * H; ++c) acc[r][c] = Num<T>::acc_init();

  // kStages-deep pipeline with one barrier per chunk: after the barrier of chunk ch every warp
  // is past chunk ch-1, so chunk ch + kStages - 1 is issued into that stage.
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s)
    if (s < nch) load_chunk(s, s * kBK);
  for (int ch = 0; ch < nch; ++ch) {
    if (nch - 1 - ch >= kStages - 2) cp_async_wait<kStages - 2>();   // chunk ch has landed
    else cp_async_wait<0>();
    __syncthreads();
    if (ch + kStages - 1 < nch) load_chunk((ch + kStages - 1) % kStages, (ch + kStages - 1) * kBK);
    if (ch == nch - 1 && src->old) {
      // the last chunk: the other stages are free — stage the tile's current values there (one
      // contiguous TM x TN block from stage (ch+1) % kStages on; the caller guarantees it fits
      // and does not wrap), so the epilogue compares against shared memory instead of waiting
      // on one L2 round trip per row (its long-scoreboard stall, ncu at C2)
      T *dst = smem + ((ch + 1) % kStages) * S::kStage;
      int tv;
      asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tv));
      const T *o = src->old;
      const int64_t ldo = src->ldo;
#pragma unroll 4
      for (int e = tv; e < TM * TN / 4; e += kThreads) {
        const int r = e / (TN / 4), c = (e % (TN / 4)) * 4;
        cp_async16(dst + r * TN + c, o + (int64_t)r * ldo + c);
      }
      cp_async_commit();
    }
    const T *as = smem + (ch % kStages) * S::kStage + ty * S::AS;
    const T *bs = smem + (ch % kStages) * S::kStage + S::kA + tx * 4;
#pragma unroll
    for (int q = 0; q < kBK / 4; ++q) {
      V b[4][H];   // b[k][h] = B[4q+k][4tx + 4TX*h .. +3]
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int h = 0; h < H; ++h)
          b[k][h] = *reinterpret_cast<const V *>(bs + (4 * q + k) * S::BSTR + 4 * TX * h);
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        const V a = *reinterpret_cast<const V *>(as + TY * r * S::AS + 4 * q);
        // k-pair outer, column group inner: consecutive FMNMX3 on one accumulator are
        // H*4 instructions apart (hides the FADD2 -> FMNMX3 -> FMNMX3 latency chain)
#pragma unroll
        for (int h = 0; h < H; ++h) {
          T *x = &acc[r][4 * h];
          relax2k(x[0], x[1], x[2], x[3], a.x, a.y, b[0][h], b[1][h]);
        }
#pragma unroll
        for (int h = 0; h < H; ++h) {
          T *x = &acc[r][4 * h];
          relax2k(x[0], x[1], x[2], x[3], a.z, a.w, b[2][h], b[3][h]);
        }
      }
    }
  }
}

// Epilogue of one tile: strict improvements only ("one comparison"); 16-B stores of the
// changed vectors, P written for changed elements (KEY: the arg-min k = kgrp + the key's k code;
// TAG: `tag`). Rows in [mr_lo, mr_hi) and columns in [mc_lo, mc_hi) are left alone. CG: read
// the old tile through L2 (.cg) — the persistent kernel's tiles are written by other SMs, whose
// lines this SM's L1 may hold stale. Returns the largest stored key (KEY), else 0.
template <typename T, int TM, int TN, int MODE, bool CG = false>
__device__ __forceinline__ int tile_epilogue(T *__restrict__ D, int32_t *__restrict__ P, int64_t ld, int i0,
                                             int j0, int mr_lo, int mr_hi, int mc_lo, int mc_hi, int tag,
                                             int kgrp,
                                             const T (&acc)[TileShape<TM, TN>::RM][4 * TileShape<TM, TN>::H],
                                             const T *old_s = nullptr) {
  using S = TileShape<TM, TN>;
  using V = typename Vec4<T>::V;
  constexpr int RM = S::RM, H = S::H, TX = S::TX, TY = S::TY;
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  int kmax = 0;
#pragma unroll
  for (int r = 0; r < RM; ++r) {
    const int i = i0 + ty + TY * r;
    const bool row_ok = !(i >= mr_lo && i < mr_hi);
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int jb = j0 + 4 * tx + 4 * TX * h;
      V *dp = reinterpret_cast<V *>(D + (int64_t)i * ld + jb);
      V old;
      if (old_s) old = *reinterpret_cast<const V *>(old_s + (ty + TY * r) * TN + 4 * tx + 4 * TX * h);
      else if constexpr (CG) old = __ldcg(dp);
      else old = *dp;
      V nv = old;
      bool any = false;
      int32_t pv[4];
      bool chg[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = jb + e;
        const T m = acc[r][4 * h + e];
        chg[e] = row_ok && !(j >= mc_lo && j < mc_hi) && m < (T)vget(old, e);
        pv[e] = tag;
        if (chg[e]) {
          any = true;
          if (is_key(MODE)) {
            const int kk = Num<T>::lowk(m - Num<T>::from_int(j & kKeyMask));   // arg-min k & kKeyMask
            const T key = m - Num<T>::from_int(kk);
            vset(nv, e, key);
            kmax = max(kmax, Num<T>::bits(key));
            pv[e] = kgrp + kk;
          } else {
            vset(nv, e, m);
          }
        }
      }
      if (any) {
        *dp = nv;
        if (MODE != MODE_PLAIN) {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (chg[e]) P[(int64_t)i * ld + jb + e] = pv[e];
        }
      }
    }
  }
  return kmax;
}

// ---------------------------------------------------------------------------------
// Min-plus tile kernel (phases 2 and 3). Tile origin (i0, j0) = (row0 + by*TM, col0 + bx*TN);
// blockIdx.z selects one of two strip descriptions (phase 2 launches both strips at once).
//   D[i][j] <- min(D[i][j], min_{k<Kd} D[i][kb+k] + B[k][j])
// with i a LOCAL row of this GPU's block-row partition (all rows on one GPU) and B the pivot
// row strip (rows kb..kb+Kd of the global matrix: in D on its owner, the broadcast buffer
// elsewhere), for the tile's (i,j), excluding rows in [mr_lo, mr_hi) and columns in [mc_lo, mc_hi)
// (strips owned by other phases). In-place use (phase 2: the tile is its own A or B)
// is safe: a CTA reads all its A/B chunks before its epilogue writes, and no other CTA writes
// what it reads.
// The main loop and the epilogue are written out here rather than calling tile_mainloop /
// tile_epilogue (the same arithmetic, used by the persistent kernel): with the calls, ptxas
// spills 20 B of cp.async addresses at the 128-register cap and reloads them every k-chunk,
// which cost 6% of the C4 solve (39.8 -> 37.4 TFLOPS, profiles/r02_refactor_regression.json).
template <typename T, int TM, int TN, int MODE, bool DUAL = false>
__global__ void __launch_bounds__(kThreads, TileShape<TM, TN>::kMinBlocks)
minplus_tile_kernel(T *__restrict__ D, int32_t *__restrict__ P, const TileArgs g, int *maxkey) {
  using S = TileShape<TM, TN>;
  using V = typename Vec4<T>::V;
  constexpr int RM = S::RM, H = S::H, TX = S::TX, TY = S::TY;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *smem = reinterpret_cast<T *>(smem_raw);

  // tile origin and exclusions (computed again after the main loop: see the epilogue)
  // colstrip 2 / colstep (pairs of plain rounds) never occur with round tags: compiled out there
  constexpr bool PAIRS = MODE != MODE_TAG;
  const int cstrip = g.colstrip;
  // a launch that follows this one with programmatic serialization (the next pair's bulk
  // launch) may start its CTAs once every CTA of this one has started; it
  // waits for this grid's completion only before its own epilogue (griddepcontrol.wait below)
  asm volatile("griddepcontrol.launch_dependents;");
  const TileSlot ts = tile_slot<TM, TN, DUAL, PAIRS>(g, blockIdx.x, blockIdx.y, blockIdx.z);
  if (ts.skip) return;
  const int i0 = ts.i0, j0 = ts.j0;

  const int64_t ld = g.ld;
  const int kb = PAIRS ? (cstrip ? (cstrip == 2 ? (j0 ^ 128) : j0) : g.kb) : (g.colstrip ? j0 : g.kb);
  // TAG / PLAIN: the cp.async source addresses are recomputed every chunk from the tile origin in
  // shared memory and a fresh %tid.x, so no address lives across the main loop — with the two
  // 64-bit source pointers live, ptxas spilled them (20 B) and reloaded them after every
  // chunk's barrier, the same pattern that cost the KEY variant 6% when it appeared there
  // (profiles/r02_refactor_regression.json). The KEY variant allocates spill-free as it is.
  __shared__ int s_org[4];
  if constexpr (MODE != MODE_KEY) {
    if (threadIdx.x == 0) {
      s_org[0] = i0;
      s_org[1] = j0;
      s_org[2] = kb;
      s_org[3] = cstrip;
    }
    __syncthreads();
  }
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  // Warm L2 with this tile of D for the epilogue's compare (128-B lines, per-thread
  // addresses): the tile is read once per round from HBM, and its latency was the
  // epilogue's top stall.
  {
    constexpr int LPR = TN * (int)sizeof(T) / 128;   // lines per tile row
    for (int l = tid; l < TM * LPR; l += kThreads)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(D + (int64_t)(i0 + l / LPR) * ld + j0 + (l % LPR) * (128 / (int)sizeof(T))));
  }

  // cp.async assignments: A chunk TM x kBK, B chunk kBK x TN, 16 B per copy.
  constexpr int A_PER = TM * (kBK / 4) / kThreads;
  constexpr int A_ROWS = kThreads / (kBK / 4);
  constexpr int B_PER = kBK * (TN / 4) / kThreads;
  constexpr int B_ROWS = kThreads / (TN / 4);
  static_assert(A_PER >= 1 && B_PER >= 1, "copy mapping");
  const int a_r = tid / (kBK / 4), a_c = (tid % (kBK / 4)) * 4;
  const int b_r = tid / (TN / 4), b_c = (tid % (TN / 4)) * 4;
  const T *a_src = D + (int64_t)(i0 + a_r) * ld + kb + a_c;
  const int64_t ldb = g.ldb;
  const T *b_src = static_cast<const T *>(g.B) + (int64_t)((cstrip ? kb : 0) + b_r) * ldb + j0 + b_c;

  auto load_chunk = [&](int stage, int k0) {
    T *as = smem + stage * S::kStage;
    T *bs = as + S::kA;
    if constexpr (MODE == MODE_KEY) {
#pragma unroll
      for (int t = 0; t < A_PER; ++t)
        cp_async16(as + (a_r + t * A_ROWS) * S::AS + a_c, a_src + k0 + (int64_t)t * A_ROWS * ld);
#pragma unroll
      for (int t = 0; t < B_PER; ++t)
        cp_async16(bs + (b_r + t * B_ROWS) * S::BSTR + b_c, b_src + (int64_t)(k0 + t * B_ROWS) * ldb);
    } else {
      int tv;
      asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tv));
      const int oi = s_org[0], oj = s_org[1], okb = s_org[2], ocs = s_org[3];
      const int ar = tv / (kBK / 4), ac = (tv % (kBK / 4)) * 4, br = tv / (TN / 4), bc = (tv % (TN / 4)) * 4;
      const T *asrc = D + (int64_t)(oi + ar) * ld + okb + ac;
      const T *bsrc = static_cast<const T *>(g.B) + (int64_t)((ocs ? okb : 0) + br) * ldb + oj + bc;
#pragma unroll
      for (int t = 0; t < A_PER; ++t)
        cp_async16(as + (ar + t * A_ROWS) * S::AS + ac, asrc + k0 + (int64_t)t * A_ROWS * ld);
#pragma unroll
      for (int t = 0; t < B_PER; ++t)
        cp_async16(bs + (br + t * B_ROWS) * S::BSTR + bc, bsrc + (int64_t)(k0 + t * B_ROWS) * ldb);
    }
    cp_async_commit();
  };

  T acc[RM][4 * H];
#pragma unroll
  for (int r = 0; r < RM; ++r)
#pragma unroll
    for (int c = 0; c < 4 * H; ++c) acc[r][c] = Num<T>::acc_init();

  // kStages-deep pipeline with one barrier per chunk: after the barrier of chunk ch every warp
  // is past chunk ch-1, so chunk ch + kStages - 1 is issued into that stage.
  const int nch = g.Kd / kBK;
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s)
    if (s < nch) load_chunk(s, s * kBK);
  for (int ch = 0; ch < nch; ++ch) {
    if (nch - 1 - ch >= kStages - 2) cp_async_wait<kStages - 2>();   // chunk ch has landed
    else cp_async_wait<0>();
    __syncthreads();
    if (ch + kStages - 1 < nch) load_chunk((ch + kStages - 1) % kStages, (ch + kStages - 1) * kBK);
    const T *as = smem + (ch % kStages) * S::kStage + ty * S::AS;
    const T *bs = smem + (ch % kStages) * S::kStage + S::kA + tx * 4;
#pragma unroll
    for (int q = 0; q < kBK / 4; ++q) {
      V b[4][H];   // b[k][h] = B[4q+k][4tx + 4TX*h .. +3]
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int h = 0; h < H; ++h)
          b[k][h] = *reinterpret_cast<const V *>(bs + (4 * q + k) * S::BSTR + 4 * TX * h);
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        const V a = *reinterpret_cast<const V *>(as + TY * r * S::AS + 4 * q);
        // k-pair outer, column group inner: consecutive FMNMX3 on one accumulator are
        // H*4 instructions apart (hides the FADD2 -> FMNMX3 -> FMNMX3 latency chain)
#pragma unroll
        for (int h = 0; h < H; ++h) {
          T *x = &acc[r][4 * h];
          relax2k(x[0], x[1], x[2], x[3], a.x, a.y, b[0][h], b[1][h]);
        }
#pragma unroll
        for (int h = 0; h < H; ++h) {
          T *x = &acc[r][4 * h];
          relax2k(x[0], x[1], x[2], x[3], a.z, a.w, b[2][h], b[3][h]);
        }
      }
    }
  }

  // ---- epilogue: strict improvements only ("one comparison"); 16-B stores ----------
  // (launched with programmatic serialization: the previous launch in the stream, which wrote
  // this tile, must be complete before the tile is read and written; a no-op otherwise)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const TileSlot te = tile_slot<TM, TN, DUAL, PAIRS>(g, ctaid(0), ctaid(1), ctaid(2));
  const int mr_lo = te.mr_lo, mr_hi = te.mr_hi, mc_lo = te.mc_lo, mc_hi = te.mc_hi;
  const int kgrp = (g.colstrip ? te.j0 : g.kb) & ~kKeyMask;
  const int tag = PAIRS ? (cstrip ? (cstrip == 2 ? (te.j0 ^ 128) : te.j0) >> 7 : g.tag) : (g.colstrip ? te.j0 >> 7 : g.tag);
  int kmax = 0;
#pragma unroll
  for (int r = 0; r < RM; ++r) {
    const int i = te.i0 + ty + TY * r;
    const bool row_ok = !(i >= mr_lo && i < mr_hi);
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int jb = te.j0 + 4 * tx + 4 * TX * h;
      V *dp = reinterpret_cast<V *>(D + (int64_t)i * g.ld + jb);
      const V old = *dp;
      V nv = old;
      bool any = false;
      int32_t pv[4];
      bool chg[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = jb + e;
        const T m = acc[r][4 * h + e];
        chg[e] = row_ok && !(j >= mc_lo && j < mc_hi) && m < (T)vget(old, e);
        pv[e] = tag;
        if (chg[e]) {
          any = true;
          if (is_key(MODE)) {
            const int kk = Num<T>::lowk(m - Num<T>::from_int(j & kKeyMask));   // arg-min k & kKeyMask
            const T key = m - Num<T>::from_int(kk);
            vset(nv, e, key);
            kmax = max(kmax, Num<T>::bits(key));
            pv[e] = kgrp + kk;
          } else {
            vset(nv, e, m);
          }
        }
      }
      if (any) {
        *dp = nv;
        if (MODE != MODE_PLAIN) {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (chg[e]) P[(int64_t)i * g.ld + jb + e] = pv[e];
        }
      }
    }
  }
  if (is_key(MODE)) {
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    if ((tid & 31) == 0 && kmax > 0) atomicMax(maxkey, kmax);
  }
  if (!DUAL && TM == 128 && TN == 128 && g.order && (int)blockIdx.x < g.nprio) {
    __threadfence();                       // this CTA's D / P stores before the count
    __syncthreads();
    if (tid == 0) atomicAdd(g.done, 1);
  }
}

// Look-ahead gate: the pivot stream waits until `target` look-ahead tiles of the running
// ordered phase-3 launch have been stored (one thread; acquire load + back-off). Bounded: after
// timeout_ns of global time it sets bit 4 of *flags (the host fails the solve) and returns, so
// an aborted or never-scheduled producer cannot hang the stream.
__global__ void wait_count_kernel(const int *done, int target, int *flags, unsigned long long timeout_ns) {
  int v;
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(done) : "memory");
    if (v >= target) break;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      atomicOr(flags, 16);
      break;
    }
    __nanosleep(256);
  }
}

// Phase 1, two steps per barrier: columns c, c+1 of one row relaxed through k and k+1
// (candidates a0 + b0*, a1 + b1*): FADD2 + FMNMX3 (FP32) or VIADDMNMX (INT32).
__device__ __forceinline__ void relax_pair2(float &x0, float &x1, float a0, float a1, float b00, float b01,
                                            float b10, float b11) {
  const float2 s0 = __fadd2_rn(make_float2(a0, a0), make_float2(b00, b01));
  const float2 s1 = __fadd2_rn(make_float2(a1, a1), make_float2(b10, b11));
  x0 = fminf(x0, fminf(s0.x, s1.x));
  x1 = fminf(x1, fminf(s0.y, s1.y));
}
__device__ __forceinline__ void relax_pair2(int &x0, int &x1, int a0, int a1, int b00, int b01, int b10,
                                            int b11) {
  x0 = __viaddmin_s32(a0, b00, x0);
  x0 = __viaddmin_s32(a1, b10, x0);
  x1 = __viaddmin_s32(a0, b01, x1);
  x1 = __viaddmin_s32(a1, b11, x1);
}
__device__ __forceinline__ float tmin(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ int tmin(int a, int b) { return min(a, b); }

// ---------------------------------------------------------------------------------
// Phase 1: closure of the diagonal block D_KK in shared memory. For each k of the
// block in order: d[a][b] = min(d[a][b], d[a][k] + d[k][b]) (strict '<'). Row k and column k
// are invariant during step k because d[k][k] = 0, so one barrier per k is exact.
// 1024 threads; thread (tx, ty) owns the R x R elements a = R*ty + r, b = R*tx + c in
// registers (R = BS/32). Step k reads row k from sD and column k from its transposed copy
// sDT (one vector load each); the owners of row k+1 and column k+1 publish them to shared
// memory before the barrier, so no other element needs mirroring.
// Key mode: candidate (d'[a][k] - (k&255)) + d'[k][b] = S*256 + (b&255) is directly the new
// key when S < D, so min() keeps keys exact; P[a][b] <- k (last improving k) on change.
// R consecutive values of shared memory into registers with the widest aligned vector loads.
template <typename T, int R>
__device__ __forceinline__ void lds_vec(T (&out)[R], const T *src) {
  if constexpr (R % 4 == 0) {
    using V = typename Vec4<T>::V;
#pragma unroll
    for (int q = 0; q < R / 4; ++q) {
      const V v = reinterpret_cast<const V *>(src)[q];
      out[4 * q] = v.x; out[4 * q + 1] = v.y; out[4 * q + 2] = v.z; out[4 * q + 3] = v.w;
    }
  } else if constexpr (R == 2) {
    using V2 = typename std::conditional<Num<T>::kIsInt, int2, float2>::type;
    const V2 v = *reinterpret_cast<const V2 *>(src);
    out[0] = v.x; out[1] = v.y;
  } else {
#pragma unroll
    for (int q = 0; q < R; ++q) out[q] = src[q];
  }
}

// R consecutive values of global memory into registers (vector loads); CG: through L2 (.cg),
// for tiles other SMs wrote (the persistent kernel: this SM's L1 may hold stale lines).
template <typename T, int R, bool CG>
__device__ __forceinline__ void ldg_vec(T (&out)[R], const T *src) {
  if constexpr (!CG) {
    lds_vec<T, R>(out, src);
  } else if constexpr (R % 4 == 0) {
    using V = typename Vec4<T>::V;
#pragma unroll
    for (int q = 0; q < R / 4; ++q) {
      const V v = __ldcg(reinterpret_cast<const V *>(src) + q);
      out[4 * q] = v.x; out[4 * q + 1] = v.y; out[4 * q + 2] = v.z; out[4 * q + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < R; ++q) out[q] = __ldcg(src + q);
  }
}
template <bool CG, typename T> __device__ __forceinline__ T ldg1(const T *p) {
  if constexpr (CG) return __ldcg(p);
  else return *p;
}

// Shared memory of the phase-1 bodies (rows / columns k, k+1 double-buffered): 4 KB at BS = 128.
template <typename T, int BS> struct P1Smem {
  using T2 = typename std::conditional<Num<T>::kIsInt, int2, float2>::type;
  __align__(16) T rowb[2][2][BS];
  __align__(16) T2 colb[2][BS];
};

template <typename T, int BS, int MODE, int NT = kP1Side, bool CG = false>
__device__ __forceinline__ void phase1_body(T *__restrict__ D, int32_t *__restrict__ P, int64_t ld, int r0,
                                            int kb, int tag, int *maxkey, P1Smem<T, BS> &sm) {
  constexpr int R = BS / NT;
  static_assert(R % 2 == 0, "step parity = register slot parity needs an even R");
  // row k and column k of the current step, double-buffered by step parity (2 KB at BS = 128)
  T (*rowb)[BS] = sm.rowb[0];
  T (*colb)[BS] = sm.rowb[1];
  const int tx = threadIdx.x % NT, ty = threadIdx.x / NT;
  T *Dk = D + (int64_t)r0 * ld + kb;                // D_KK: local row r0, global column kb
  int32_t *Pk = P ? P + (int64_t)r0 * ld + kb : nullptr;
  T d[R][R];
  int32_t p[R][R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    ldg_vec<T, R, CG>(d[r], Dk + (int64_t)(R * ty + r) * ld + R * tx);   // 16-B global loads
#pragma unroll
    for (int c = 0; c < R; ++c) p[r][c] = -1;
  }
  if (ty == 0) {
#pragma unroll
    for (int c = 0; c < R; ++c) rowb[0][R * tx + c] = d[0][c];
  }
  if (tx == 0) {
#pragma unroll
    for (int r = 0; r < R; ++r) colb[0][R * ty + r] = d[r][0];
  }
  __syncthreads();
  // k is unrolled by R so that "row/column k+1 lives in register slot (k+1) % R" is a
  // compile-time index (a runtime index into d[][] would spill the register array)
  for (int k0 = 0; k0 < BS; k0 += R) {
#pragma unroll
    for (int kr = 0; kr < R; ++kr) {
      const int k = k0 + kr, buf = kr & 1;       // R is even: k & 1 == kr & 1
      T colv[R], rowv[R];
      lds_vec<T, R>(colv, &colb[buf][R * ty]);   // d[a][k], own rows
      lds_vec<T, R>(rowv, &rowb[buf][R * tx]);   // d[k][b], own cols
      const T kp = is_key(MODE) ? Num<T>::from_int((kb + k) & kKeyMask) : (T)0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        // exact (keys are integers < 2^24 / 2^30); INF must stay INF (INT32 sentinel arithmetic)
        const T cr = (is_key(MODE) && Num<T>::finite(colv[r])) ? colv[r] - kp : colv[r];
#pragma unroll
        for (int c = 0; c < R; ++c) {
          const T s = cr + rowv[c];
          if (is_key(MODE)) p[r][c] = s < d[r][c] ? kb + k : p[r][c];
          d[r][c] = s < d[r][c] ? s : d[r][c];
        }
      }
      // publish row k+1 and column k+1 (register slot (kr+1) % R of owner ty / tx) into the
      // other buffer; everyone finished reading it before the previous barrier
      const int slot = (kr + 1) % R;   // constant after unrolling
      const int owner = (k + 1) / R;
      if (k + 1 < BS) {
        if (owner == ty) {
#pragma unroll
          for (int c = 0; c < R; ++c) rowb[buf ^ 1][R * tx + c] = d[slot][c];
        }
        if (owner == tx) {
#pragma unroll
          for (int r = 0; r < R; ++r) colb[buf ^ 1][R * ty + r] = d[r][slot];
        }
      }
      __syncthreads();
    }
  }
  int kmax = 0;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < R; ++c) {
      const int a = R * ty + r, b = R * tx + c;
      const int64_t off = (int64_t)a * ld + b;
      if (d[r][c] < ldg1<CG>(Dk + off)) {
        Dk[off] = d[r][c];
        if (MODE == MODE_TAG) Pk[off] = tag;
        if (is_key(MODE)) {
          Pk[off] = p[r][c];
          kmax = max(kmax, Num<T>::bits(d[r][c]));
        }
      }
    }
  if (is_key(MODE)) {
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    if ((threadIdx.x & 31) == 0 && kmax > 0) atomicMax(maxkey, kmax);
  }
}

template <typename T, int BS, int MODE, int NT = kP1Side>
__global__ void __launch_bounds__(NT * NT)
phase1_kernel(T *__restrict__ D, int32_t *__restrict__ P, int64_t ld, int r0, int kb, int tag,
              int *maxkey) {
  __shared__ P1Smem<T, BS> sm;
  phase1_body<T, BS, MODE, NT>(D, P, ld, r0, kb, tag, maxkey, sm);
}

// Phase 1 for PLAIN / TAG (no per-step P), two steps per barrier: row / column k+1 are brought
// to their state after step k by every thread (col'[a] = min(col_k1[a], col_k[a] + D[k][k+1]),
// row'[b] = min(row_k1[b], D[k+1][k] + row_k[b])), then x = min(x, c_k, c'_k+1) — exactly the
// sequential loop's values (min is exact; each candidate is the same single rounded sum).
// Thread layout of the two-steps-per-barrier phase-1 bodies: RY rows x RX columns per thread,
// (BS/RY) x (BS/RX) threads (BS = 128: 256 threads of 8 x 8; 512 threads of 8 x 4 or 4 x 8 fit
// in half the register file only with spills and measured slower).
template <int BS, int RY, int RX> struct P1Layout {
  static constexpr int NX = BS / RX, NY = BS / RY, kThreads = NX * NY;
  static constexpr int U = RY > RX ? RY : RX;   // k unroll period: row / column slots compile-time
  static_assert(RY % 2 == 0 && RX % 2 == 0 && U % RY == 0 && U % RX == 0 && BS % U == 0, "phase-1 layout");
};

template <typename T, int BS, int MODE, int RY, int RX, bool CG = false>
__device__ __forceinline__ void phase1_pair_body(T *__restrict__ D, int32_t *__restrict__ P, int64_t ld, int r0,
                                                 int kb, int tag, P1Smem<T, BS> &sm) {
  using L = P1Layout<BS, RY, RX>;
  static_assert(!is_key(MODE), "pairs of steps; keyed modes use their own kernels");
  using T2 = typename std::conditional<Num<T>::kIsInt, int2, float2>::type;
  T (*rowb)[2][BS] = sm.rowb;   // rows k, k+1 (pair parity)
  T2 (*colb)[BS] = sm.colb;     // (column k, column k+1) per row
  const int tx = threadIdx.x % L::NX, ty = threadIdx.x / L::NX;
  T *Dk = D + (int64_t)r0 * ld + kb;
  T d[RY][RX];
#pragma unroll
  for (int r = 0; r < RY; ++r) ldg_vec<T, RX, CG>(d[r], Dk + (int64_t)(RY * ty + r) * ld + RX * tx);
  if (ty == 0) {
#pragma unroll
    for (int c = 0; c < RX; ++c) {
      rowb[0][0][RX * tx + c] = d[0][c];
      rowb[0][1][RX * tx + c] = d[1][c];
    }
  }
  if (tx == 0) {
#pragma unroll
    for (int r = 0; r < RY; ++r) colb[0][RY * ty + r] = T2{d[r][0], d[r][1]};
  }
  __syncthreads();
  for (int k0 = 0; k0 < BS; k0 += L::U) {
#pragma unroll
    for (int kr = 0; kr < L::U; kr += 2) {
      const int k = k0 + kr, buf = (k >> 1) & 1;
      T rk[RX], rk1[RX];
      lds_vec<T, RX>(rk, &rowb[buf][0][RX * tx]);
      lds_vec<T, RX>(rk1, &rowb[buf][1][RX * tx]);
      const T d01 = rowb[buf][0][k + 1];   // D[k][k+1]
      const T d10 = colb[buf][k + 1].x;    // D[k+1][k]
#pragma unroll
      for (int c = 0; c < RX; ++c) rk1[c] = tmin(rk1[c], d10 + rk[c]);   // INT32: <= 2 INF, no overflow
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const T2 ca = colb[buf][RY * ty + r];
        const T ck1 = tmin(ca.y, ca.x + d01);
#pragma unroll
        for (int c = 0; c < RX; c += 2)
          relax_pair2(d[r][c], d[r][c + 1], ca.x, ck1, rk[c], rk[c + 1], rk1[c], rk1[c + 1]);
      }
      if (k + 2 < BS) {   // publish rows / columns k+2, k+3 (slots of one owner: k+2 is even)
        if ((k + 2) / RY == ty) {
          const int s2 = (kr + 2) % RY, s3 = (kr + 3) % RY;
#pragma unroll
          for (int c = 0; c < RX; ++c) {
            rowb[buf ^ 1][0][RX * tx + c] = d[s2][c];
            rowb[buf ^ 1][1][RX * tx + c] = d[s3][c];
          }
        }
        if ((k + 2) / RX == tx) {
          const int s2 = (kr + 2) % RX, s3 = (kr + 3) % RX;
#pragma unroll
          for (int r = 0; r < RY; ++r) colb[buf ^ 1][RY * ty + r] = T2{d[r][s2], d[r][s3]};
        }
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int r = 0; r < RY; ++r)
#pragma unroll
    for (int c = 0; c < RX; ++c) {
      const int a = RY * ty + r, b = RX * tx + c;
      const int64_t off = (int64_t)a * ld + b;
      if (d[r][c] < ldg1<CG>(Dk + off)) {
        Dk[off] = d[r][c];
        if (MODE == MODE_TAG) P[(int64_t)(r0 + a) * ld + kb + b] = tag;
      }
    }
}


template <typename T, int BS, int MODE, int RY, int RX>
__global__ void __launch_bounds__(P1Layout<BS, RY, RX>::kThreads, 2)   // half the register file: fits beside a phase-3 CTA
phase1_pair_kernel(T *__restrict__ D, int32_t *__restrict__ P, int64_t ld, int r0, int kb, int tag) {
  __shared__ P1Smem<T, BS> sm;
  phase1_pair_body<T, BS, MODE, RY, RX>(D, P, ld, r0, kb, tag, sm);
}

// Phase 1, FP32 keyed mode, without a per-relaxation select for P. The running value of
// (a, b) is kept in the form  x = D*256 - 0.5  while unchanged, and a candidate through k is
// the integer  c_k = D[a][k]*256 + k' + D[k][b]*256  (k' = (kb + k) & 255, increasing in k
// inside a block): c_k < x  <=>  D[a][k] + D[k][b] < D (strict, P:125 / reading R2), and the
// minimum over the sequence is the smallest distance reached first, with its k in the low 7
// bits — the sequential strict-< result of the paper's loop, with one FADD + one FMNMX per
// relaxation. Row k+1 is published as D*256 (B side), column k+1 as D*256 + k' (A side), both
// recovered as floor((x + 0.5) / 256) * 256. Exact: keys < 2^23 (kKeyMaxF32), half-integers.
// core: the block at Dk (pitch ld), its P at Pk (pitch ldp); column / intermediate codes are
// klow + local index (klow + BS <= 256), P values kgrp + code.
template <int BS, int RY, int RX, bool CG = false>
__device__ __forceinline__ void phase1_key_f32_core(float *__restrict__ Dk, int64_t ld, int32_t *__restrict__ Pk,
                                                    int64_t ldp, int kgrp, int klow, int *maxkey,
                                                    P1Smem<float, BS> &sm) {
  using L = P1Layout<BS, RY, RX>;
  float (*rowb)[2][BS] = sm.rowb;   // rows k, k+1, B form D*256  (pair parity)
  float2 (*colb)[BS] = sm.colb;     // (column k, column k+1) per row, A form D*256 + k'
  const int tx = threadIdx.x % L::NX, ty = threadIdx.x / L::NX;
  float x[RY][RX];
#pragma unroll
  for (int r = 0; r < RY; ++r) {
    float key[RX];
    ldg_vec<float, RX, CG>(key, Dk + (int64_t)(RY * ty + r) * ld + RX * tx);  // D*256 + ((kb+b)&255) or +inf
#pragma unroll
    for (int c = 0; c < RX; ++c) x[r][c] = key[c] - (float)(klow + RX * tx + c) - 0.5f;   // D*256 - 0.5
  }
  // steps k and k+1 per barrier (the sequential loop's values, two steps at a time): every
  // thread brings row / column k+1 to their state after step k itself,
  //   col'[a] = min(col_k1[a], col_k[a] + D[k][k+1]*256 + 1)   ((k+1)' = k' + 1 inside the block)
  //   row'[b] = min(row_k1[b], D[k+1][k]*256 + row_k[b])
  // and folds both candidates into x with FADD2 + FMNMX3: x = min(x, c_k, c'_k+1) (min is exact,
  // every candidate is the same integer sum as in the one-step loop).
  if (ty == 0) {
#pragma unroll
    for (int c = 0; c < RX; ++c) {
      rowb[0][0][RX * tx + c] = x[0][c] + 0.5f;                           // D*256
      rowb[0][1][RX * tx + c] = x[1][c] + 0.5f;
    }
  }
  if (tx == 0) {
#pragma unroll
    for (int r = 0; r < RY; ++r)                                          // + k'
      colb[0][RY * ty + r] = make_float2(x[r][0] + 0.5f + (float)klow, x[r][1] + 0.5f + (float)(klow + 1));
  }
  __syncthreads();
  for (int k0 = 0; k0 < BS; k0 += L::U) {
#pragma unroll
    for (int kr = 0; kr < L::U; kr += 2) {
      const int k = k0 + kr, buf = (k >> 1) & 1;
      float rk[RX], rk1[RX];
      lds_vec<float, RX>(rk, &rowb[buf][0][RX * tx]);    // B side, own cols
      lds_vec<float, RX>(rk1, &rowb[buf][1][RX * tx]);
      const float d01 = rowb[buf][0][k + 1] + 1.0f;              // D[k][k+1]*256 + 1
      const float d10 = colb[buf][k + 1].x - (float)(klow + k);  // D[k+1][k]*256 (exact; inf stays)
#pragma unroll
      for (int c = 0; c < RX; ++c) rk1[c] = fminf(rk1[c], d10 + rk[c]);
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const float2 ca = colb[buf][RY * ty + r];                // A side, own row (broadcast)
        const float ck1 = fminf(ca.y, ca.x + d01);
#pragma unroll
        for (int c = 0; c < RX; c += 2)
          relax_pair2(x[r][c], x[r][c + 1], ca.x, ck1, rk[c], rk[c + 1], rk1[c], rk1[c + 1]);
      }
      // publish rows / columns k+2 and k+3 (slots of one owner: k+2 is even)
      if (k + 2 < BS) {
        if ((k + 2) / RY == ty) {
          const int s2 = (kr + 2) % RY, s3 = (kr + 3) % RY;
#pragma unroll
          for (int c = 0; c < RX; ++c) {
            rowb[buf ^ 1][0][RX * tx + c] = floorf((x[s2][c] + 0.5f) * (1.0f / kKeyMul)) * (float)kKeyMul;
            rowb[buf ^ 1][1][RX * tx + c] = floorf((x[s3][c] + 0.5f) * (1.0f / kKeyMul)) * (float)kKeyMul;
          }
        }
        if ((k + 2) / RX == tx) {
          const int s2 = (kr + 2) % RX, s3 = (kr + 3) % RX;
          const float kp = (float)(klow + k + 2);
#pragma unroll
          for (int r = 0; r < RY; ++r)
            colb[buf ^ 1][RY * ty + r] = make_float2(floorf((x[r][s2] + 0.5f) * (1.0f / kKeyMul)) * (float)kKeyMul + kp,
                                                     floorf((x[r][s3] + 0.5f) * (1.0f / kKeyMul)) * (float)kKeyMul + kp + 1.0f);
        }
      }
      __syncthreads();
    }
  }
  int kmax = 0;
#pragma unroll
  for (int r = 0; r < RY; ++r)
#pragma unroll
    for (int c = 0; c < RX; ++c) {
      const float v = x[r][c];
      if (v < __int_as_float(0x7f800000) && v == floorf(v)) {   // an integer: strictly improved
        const int a = RY * ty + r, b = RX * tx + c;
        const float hi = floorf(v * (1.0f / kKeyMul)) * (float)kKeyMul;
        const int kk = (int)(v - hi);
        const float key = hi + (float)(klow + b);
        Dk[(int64_t)a * ld + b] = key;
        Pk[(int64_t)a * ldp + b] = kgrp + kk;
        kmax = max(kmax, __float_as_int(key));
      }
    }
  kmax = __reduce_max_sync(0xffffffffu, kmax);
  if ((threadIdx.x & 31) == 0 && kmax > 0) atomicMax(maxkey, kmax);
}

template <int BS, int RY, int RX, bool CG = false>
__device__ __forceinline__ void phase1_key_f32_body(float *__restrict__ D, int32_t *__restrict__ P, int64_t ld,
                                                    int r0, int kb, int *maxkey, P1Smem<float, BS> &sm) {
  phase1_key_f32_core<BS, RY, RX, CG>(D + (int64_t)r0 * ld + kb, ld, P + (int64_t)r0 * ld + kb, ld, kb & ~kKeyMask,
                                      kb & kKeyMask, maxkey, sm);
}

template <int BS, int RY, int RX>
__global__ void __launch_bounds__(P1Layout<BS, RY, RX>::kThreads, 2)   // half the register file: fits beside a phase-3 CTA
phase1_key_f32_kernel(float *__restrict__ D, int32_t *__restrict__ P, int64_t ld, int r0, int kb,
                      int *maxkey) {
  __shared__ P1Smem<float, BS> sm;
  phase1_key_f32_body<BS, RY, RX>(D, P, ld, r0, kb, maxkey, sm);
}

// ---------------------------------------------------------------------------------
// Phase 1, blocked (PLAIN / TAG, BS = 128, 256 threads): the closure of D_KK computed as the
// paper's own blocked Floyd–Warshall one level down (P:101-112 applied to the 128 x 128 block
// with 32 x 32 sub-blocks), instead of 128 sequential steps of the whole CTA. For each
// sub-round s of 4:
//   (a) closure of the diagonal sub-block (s, s): phase1_pair_body on the 32 x 32 sub-block in
//       shared memory (256 threads of 2 x 2, 16 barriers);
//   (b) the row / column sub-strips (s, t), (t, s) as min-plus products with the closed
//       sub-block (reading R7): 128 threads each;
//   (c) the other 9 sub-blocks (t, u) <- min(., (t, s) (x) (s, u)): 256 threads of 6 x 6.
// Same distances as the sequential loop (R7, R8: min is exact, every candidate one rounded
// add). The 128 x 128 block lives in shared memory (pitch 132: conflict-free 16-B row reads
// by consecutive lanes), 69 KB: one CTA still fits beside a phase-3 CTA.
constexpr int kP1BPitch = 132;
template <typename T> struct P1BSmem {
  __align__(16) T t[128 * kP1BPitch];
  __align__(16) T rb[2][2][32];   // sub-phase (a), keyed: rows k, k+1 by pair parity
  P1Smem<T, 32> p1;               // sub-phase (a), plain: the pair-step body on the sub-block
};

// x[r][2p + e] = min(x, min_k A(r, k) + B(k, 2p + e)) over 32 k: A rows at a[r] (k contiguous),
// B column pairs at b[p] (row pitch kP1BPitch). FADD2 + FMNMX3 over two k per instruction pair.
template <typename T, int RY, int NP>
__device__ __forceinline__ void p1b_product(T (&x)[RY][2 * NP], const T *sm, const int (&a)[RY], const int (&b)[NP]) {
  using V = typename Vec4<T>::V;
  using T2 = typename std::conditional<Num<T>::kIsInt, int2, float2>::type;
#pragma unroll
  for (int k = 0; k < 32; k += 4) {
    V av[RY];
#pragma unroll
    for (int r = 0; r < RY; ++r) av[r] = *reinterpret_cast<const V *>(sm + a[r] + k);
#pragma unroll
    for (int kk = 0; kk < 4; kk += 2) {
      T2 b0[NP], b1[NP];
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        b0[q] = *reinterpret_cast<const T2 *>(sm + b[q] + (k + kk) * kP1BPitch);
        b1[q] = *reinterpret_cast<const T2 *>(sm + b[q] + (k + kk + 1) * kP1BPitch);
      }
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const T a0 = kk ? av[r].z : av[r].x, a1 = kk ? av[r].w : av[r].y;
#pragma unroll
        for (int q = 0; q < NP; ++q) relax_pair2(x[r][2 * q], x[r][2 * q + 1], a0, a1, b0[q].x, b0[q].y, b1[q].x, b1[q].y);
      }
    }
  }
}

// index g in [0, 96) of the three sub-blocks other than s -> tile index in [0, 128)
__device__ __forceinline__ int p1b_other(int g, int s) {
  const int q = g >> 5;
  return ((q < s ? q : q + 1) << 5) + (g & 31);
}

template <typename T, int MODE, bool CG = false>
__device__ __forceinline__ void phase1_blocked_body(T *__restrict__ D, int32_t *__restrict__ P, int64_t ld, int r0,
                                                    int kb, int tag, P1BSmem<T> &sm) {
  static_assert(!is_key(MODE), "plain distances / round tags");
  using V = typename Vec4<T>::V;
  T *t = sm.t;
  const int tid = threadIdx.x;
  T *Dk = D + (int64_t)r0 * ld + kb;
  for (int e = tid; e < 128 * 32; e += 256) {   // the block into shared memory (16-B loads)
    const int r = e >> 5, c4 = (e & 31) * 4;
    V v;
    if constexpr (CG) v = __ldcg(reinterpret_cast<const V *>(Dk + (int64_t)r * ld + c4));
    else v = *reinterpret_cast<const V *>(Dk + (int64_t)r * ld + c4);
    *reinterpret_cast<V *>(t + r * kP1BPitch + c4) = v;
  }
  __syncthreads();
  for (int s = 0; s < 4; ++s) {
    const int o = s * 32;
    // (a) closure of sub-block (s, s): the two-steps-per-barrier body on the 32 x 32 sub-block in
    //     shared memory, 256 threads of 2 x 2 (16 barriers; one warp alone measured 64 us per
    //     phase 1 against 40 for the unblocked kernel — every latency exposed)
    phase1_pair_body<T, 32, MODE_PLAIN, 2, 2, false>(t, nullptr, kP1BPitch, o, o, 0, sm.p1);
    __syncthreads();
    // (b) row sub-strips (s, t) = S* (x) (s, t) [threads 0..127: 4 rows x 3 column pairs] and
    //     column sub-strips (t, s) = (t, s) (x) S* [threads 128..255: 6 rows x 2 column pairs];
    //     every operand is read before the barrier, the results stored after it (in place)
    {
      T xr[6][6];
      int nr = 0, np = 0, orow[6], ocol[3];
      if (tid < 128) {
        const int ry = tid >> 4, cx = tid & 15;   // 8 row groups x 16 column groups
        int a[4], b[3];
#pragma unroll
        for (int r = 0; r < 4; ++r) { orow[r] = o + 4 * ry + r; a[r] = orow[r] * kP1BPitch + o; }
#pragma unroll
        for (int q = 0; q < 3; ++q) { ocol[q] = p1b_other(6 * cx + 2 * q, s); b[q] = o * kP1BPitch + ocol[q]; }
        T x4[4][6];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 6; ++c) x4[r][c] = t[orow[r] * kP1BPitch + ocol[c >> 1] + (c & 1)];
        p1b_product<T, 4, 3>(x4, t, a, b);
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 6; ++c) xr[r][c] = x4[r][c];
        nr = 4;
        np = 3;
      } else {
        const int u = tid - 128, ry = u >> 3, cx = u & 7;   // 16 row groups x 8 column groups
        int a[6], b[2];
#pragma unroll
        for (int r = 0; r < 6; ++r) { orow[r] = p1b_other(6 * ry + r, s); a[r] = orow[r] * kP1BPitch + o; }
#pragma unroll
        for (int q = 0; q < 2; ++q) { ocol[q] = o + 4 * cx + 2 * q; b[q] = o * kP1BPitch + ocol[q]; }
        T x6[6][4];
#pragma unroll
        for (int r = 0; r < 6; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) x6[r][c] = t[orow[r] * kP1BPitch + ocol[c >> 1] + (c & 1)];
        p1b_product<T, 6, 2>(x6, t, a, b);
#pragma unroll
        for (int r = 0; r < 6; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) xr[r][c] = x6[r][c];
        nr = 6;
        np = 2;
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = 0; c < 6; ++c)
          if (r < nr && (c >> 1) < np) t[orow[r] * kP1BPitch + ocol[c >> 1] + (c & 1)] = xr[r][c];
    }
    __syncthreads();
    // (c) the 9 other sub-blocks (t, u) <- min(., (t, s) (x) (s, u)): 16 x 16 threads of 6 rows x 3
    //     column pairs; each output is read and written by its own thread only
    {
      const int ry = tid >> 4, cx = tid & 15;
      int orow[6], ocol[3], a[6], b[3];
#pragma unroll
      for (int r = 0; r < 6; ++r) { orow[r] = p1b_other(6 * ry + r, s); a[r] = orow[r] * kP1BPitch + o; }
#pragma unroll
      for (int q = 0; q < 3; ++q) { ocol[q] = p1b_other(6 * cx + 2 * q, s); b[q] = o * kP1BPitch + ocol[q]; }
      T x[6][6];
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = 0; c < 6; ++c) x[r][c] = t[orow[r] * kP1BPitch + ocol[c >> 1] + (c & 1)];
      p1b_product<T, 6, 3>(x, t, a, b);
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = 0; c < 6; ++c) t[orow[r] * kP1BPitch + ocol[c >> 1] + (c & 1)] = x[r][c];
    }
    __syncthreads();
  }
  // strict improvements only: the changed elements and, TAG, their round
  for (int e = tid; e < 128 * 128; e += 256) {
    const int r = e >> 7, c = e & 127;
    const T v = t[r * kP1BPitch + c];
    if (v < ldg1<CG>(Dk + (int64_t)r * ld + c)) {
      Dk[(int64_t)r * ld + c] = v;
      if (MODE == MODE_TAG) P[(int64_t)(r0 + r) * ld + kb + c] = tag;
    }
  }
}

// Phase 1, blocked, FP32 keyed mode (the stored values are keys D*256 + (column & 255), DESIGN.md
// §4.3). (a) is phase1_key_f32_core (the select-free pair-step algebra: x = D*256 - 0.5 while
// unchanged, a candidate through k the integer D[a][k]*256 + k' + D[k][b]*256) on the sub-block
// in shared memory. (b) and (c) are products on the keys themselves: a candidate key sum is
// (D_ak + D_kb)*256 + k' + b', so the minimum with the old key D_ab*256 + b' is the smallest
// distance and, among ties, the smallest k, and it is below the old key iff strictly shorter
// (the tile epilogue's rule). Every improvement writes P (its last write is the final value).
template <bool CG = false>
__device__ __forceinline__ void phase1_blocked_key_body(float *__restrict__ D, int32_t *__restrict__ P, int64_t ld,
                                                        int r0, int kb, int *maxkey, P1BSmem<float> &sm) {
  float *t = sm.t;
  const int tid = threadIdx.x, lane = tid & 31;
  const int kgrp = kb & ~kKeyMask, klow = kb & kKeyMask;
  float *Dk = D + (int64_t)r0 * ld + kb;
  int32_t *Pk = P + (int64_t)r0 * ld + kb;
  int kmax = 0;
  for (int e = tid; e < 128 * 32; e += 256) {
    const int r = e >> 5, c4 = (e & 31) * 4;
    float4 v;
    if constexpr (CG) v = __ldcg(reinterpret_cast<const float4 *>(Dk + (int64_t)r * ld + c4));
    else v = *reinterpret_cast<const float4 *>(Dk + (int64_t)r * ld + c4);
    *reinterpret_cast<float4 *>(t + r * kP1BPitch + c4) = v;
  }
  __syncthreads();
  // keyed epilogue of one product output (row, col of the tile): store the new key, record P
  auto settle = [&](int row, int col, float m) {
    const float old = t[row * kP1BPitch + col];
    if (m < old) {
      const int kk = ((int)(m - (float)(klow + col))) & kKeyMask;   // the arg-min's k code
      const float key = m - (float)kk;
      t[row * kP1BPitch + col] = key;
      Pk[(int64_t)row * ld + col] = kgrp + kk;
      kmax = max(kmax, __float_as_int(key));
    }
  };
  for (int s = 0; s < 4; ++s) {
    const int o = s * 32;
    // (a): the select-free keyed pair-step body on the 32 x 32 sub-block in shared memory, 256
    //     threads of 2 x 2; codes klow + o + local index, P into the block's rows in global memory
    phase1_key_f32_core<32, 2, 2, false>(t + o * kP1BPitch + o, kP1BPitch, Pk + (int64_t)o * ld + o, ld, kgrp,
                                         klow + o, maxkey, sm.p1);
    __syncthreads();
    {   // (b) row sub-strips [threads 0..127: 4 rows x 3 column pairs], column sub-strips [6 x 2]
      float xr[6][6];
      int nr = 0, np = 0, orow[6], ocol[3];
      if (tid < 128) {
        const int ry = tid >> 4, cx = tid & 15;
        int a[4], b[3];
#pragma unroll
        for (int r = 0; r < 4; ++r) { orow[r] = o + 4 * ry + r; a[r] = orow[r] * kP1BPitch + o; }
#pragma unroll
        for (int q = 0; q < 3; ++q) { ocol[q] = p1b_other(6 * cx + 2 * q, s); b[q] = o * kP1BPitch + ocol[q]; }
        float x4[4][6];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 6; ++c) x4[r][c] = t[orow[r] * kP1BPitch + ocol[c >> 1] + (c & 1)];
        p1b_product<float, 4, 3>(x4, t, a, b);
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 6; ++c) xr[r][c] = x4[r][c];
        nr = 4;
        np = 3;
      } else {
        const int u = tid - 128, ry = u >> 3, cx = u & 7;
        int a[6], b[2];
#pragma unroll
        for (int r = 0; r < 6; ++r) { orow[r] = p1b_other(6 * ry + r, s); a[r] = orow[r] * kP1BPitch + o; }
#pragma unroll
        for (int q = 0; q < 2; ++q) { ocol[q] = o + 4 * cx + 2 * q; b[q] = o * kP1BPitch + ocol[q]; }
        float x6[6][4];
#pragma unroll
        for (int r = 0; r < 6; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) x6[r][c] = t[orow[r] * kP1BPitch + ocol[c >> 1] + (c & 1)];
        p1b_product<float, 6, 2>(x6, t, a, b);
#pragma unroll
        for (int r = 0; r < 6; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) xr[r][c] = x6[r][c];
        nr = 6;
        np = 2;
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = 0; c < 6; ++c)
          if (r < nr && (c >> 1) < np) settle(orow[r], ocol[c >> 1] + (c & 1), xr[r][c]);
    }
    __syncthreads();
    {   // (c) the other 9 sub-blocks
      const int ry = tid >> 4, cx = tid & 15;
      int orow[6], ocol[3], a[6], b[3];
#pragma unroll
      for (int r = 0; r < 6; ++r) { orow[r] = p1b_other(6 * ry + r, s); a[r] = orow[r] * kP1BPitch + o; }
#pragma unroll
      for (int q = 0; q < 3; ++q) { ocol[q] = p1b_other(6 * cx + 2 * q, s); b[q] = o * kP1BPitch + ocol[q]; }
      float x[6][6];
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = 0; c < 6; ++c) x[r][c] = t[orow[r] * kP1BPitch + ocol[c >> 1] + (c & 1)];
      p1b_product<float, 6, 3>(x, t, a, b);
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = 0; c < 6; ++c) settle(orow[r], ocol[c >> 1] + (c & 1), x[r][c]);
    }
    __syncthreads();
  }
  for (int e = tid; e < 128 * 128; e += 256) {   // the improved keys (P was written on the way)
    const int r = e >> 7, c = e & 127;
    const float v = t[r * kP1BPitch + c];
    if (v < ldg1<CG>(Dk + (int64_t)r * ld + c)) Dk[(int64_t)r * ld + c] = v;
  }
  kmax = __reduce_max_sync(0xffffffffu, kmax);
  if (lane == 0 && kmax > 0) atomicMax(maxkey, kmax);
}

__global__ void __launch_bounds__(256, 2)
phase1_blocked_key_kernel(float *__restrict__ D, int32_t *__restrict__ P, int64_t ld, int r0, int kb, int *maxkey) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  phase1_blocked_key_body(D, P, ld, r0, kb, maxkey, *reinterpret_cast<P1BSmem<float> *>(smem_raw));
}

template <typename T, int MODE>
__global__ void __launch_bounds__(256, 2)
phase1_blocked_kernel(T *__restrict__ D, int32_t *__restrict__ P, int64_t ld, int r0, int kb, int tag) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  phase1_blocked_body<T, MODE>(D, P, ld, r0, kb, tag, *reinterpret_cast<P1BSmem<T> *>(smem_raw));
}

// ---------------------------------------------------------------------------------
// Validation (read-only, before anything is written: fw.h error contract).
// flags: bit 0 out-of-domain value; bit 1 a finite FP32 weight is not integer-valued;
//        bit 2 an off-diagonal entry is INF (no edge). maxw: max finite off-diagonal weight
//        (INT32 value, or FP32 bit pattern — non-negative floats order like their bits).
template <typename T>
__device__ __forceinline__ void validate_one(T v, int &f, int &mx) {
  if (Num<T>::bad(v)) { f |= 1; return; }
  if (!Num<T>::finite(v)) { f |= 4; return; }
  if (!Num<T>::kIsInt && (float)v != rintf((float)v)) f |= 2;
  mx = max(mx, Num<T>::bits(v));
}

// Rows stride over (blockIdx.y, gridDim.y), columns over the x threads; 16-B vector loads when
// the rows are 16-B aligned (lds % 4 == 0 and an aligned base), a scalar tail otherwise.
template <typename T>
__global__ void validate_kernel(const T *src, int64_t lds, int64_t nrows, int64_t n, int64_t row0,
                                int *flags, int *maxw) {
  using V = typename Vec4<T>::V;
  int f = 0, mx = 0;
  const bool vec = (lds % 4 == 0) && ((uintptr_t)src % 16 == 0);
  const int64_t nv = vec ? n / 4 : 0;          // vectorised columns [0, 4 nv)
  for (int64_t i = blockIdx.y; i < nrows; i += gridDim.y) {
    const T *row = src + i * lds;
    const int64_t diag = row0 + i;               // the diagonal is overwritten with 0 (R4)
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nv;
         q += (int64_t)gridDim.x * blockDim.x) {
      const V v = reinterpret_cast<const V *>(row)[q];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (4 * q + e != diag) validate_one<T>(vget(v, e), f, mx);
    }
    for (int64_t j = 4 * nv + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x)
      if (j != diag) validate_one<T>(row[j], f, mx);
  }
  f = __reduce_or_sync(0xffffffffu, f);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) {
    if (f) atomicOr(flags, f);
    if (mx) atomicMax(maxw, mx);
  }
}

// Copy W (n x n, lds) into the padded n_pad x n_pad working matrix (ld): padded entries INF,
// diagonal 0 (R4, R11); key mode stores D*256 + (j&255). P (tags / last k) initialised to -1
// ("no intermediate yet"). src may alias D (in-place solve).
// Source value in the compute type C: identity, or INT32 -> FP32 (FW_INF_I32 -> +inf; finite
// INT32 weights below 2^24 are exact in FP32 — the host only picks FP32 compute when every
// value the solve can store stays below 2^24).
template <typename C, typename S> __device__ __forceinline__ C to_compute(S v) { return (C)v; }
template <> __device__ __forceinline__ float to_compute<float, int32_t>(int32_t v) {
  return v >= 0x3FFFFFFF ? __int_as_float(0x7f800000) : (float)v;
}

// Row loops stride by gridDim.y (grid.y is capped at 65535 rows per launch).
// src (type S) may alias D (type T, same 4-byte slots): each element is read before it is written.
template <typename T, int MODE, typename S = T>
__global__ void init_kernel(const S *src, int64_t lds, int64_t nsrc, int64_t n, int64_t row0, T *D,
                            int32_t *P, int64_t ld, int64_t n_pad, int64_t nrows) {
  // 4 consecutive elements per thread: 16-B loads of the source row when it is 16-B aligned and
  // the group lies inside the n real columns, 16-B stores of D and P (ld % 128 == 0)
  using VS = typename Vec4<S>::V;
  using VT = typename Vec4<T>::V;
  const bool vsrc = (lds % 4 == 0) && ((uintptr_t)src % 16 == 0);
  for (int64_t i = blockIdx.y; i < nrows; i += gridDim.y) {   // local row; global row0 + i
    const int64_t gi = row0 + i;
    const bool row_in = i < nsrc && gi < n;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_pad / 4;
         q += (int64_t)gridDim.x * blockDim.x) {
      const int64_t j = 4 * q;
      T v[4];
      if (row_in && vsrc && j + 4 <= n) {
        const VS s4 = *reinterpret_cast<const VS *>(src + i * lds + j);
        v[0] = to_compute<T, S>(s4.x);
        v[1] = to_compute<T, S>(s4.y);
        v[2] = to_compute<T, S>(s4.z);
        v[3] = to_compute<T, S>(s4.w);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          v[e] = (row_in && j + e < n) ? to_compute<T, S>(src[i * lds + j + e]) : Num<T>::inf();
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (gi == j + e) v[e] = 0;
        if (is_key(MODE)) v[e] = Num<T>::encode(v[e], (int)(j + e));
      }
      VT o;
      o.x = v[0]; o.y = v[1]; o.z = v[2]; o.w = v[3];
      *reinterpret_cast<VT *>(D + i * ld + j) = o;
      if (MODE != MODE_PLAIN) *reinterpret_cast<int4 *>(P + i * ld + j) = make_int4(-1, -1, -1, -1);
    }
  }
}

// FP32 compute -> INT32 storage in place (integer values below 2^24; +inf -> FW_INF_I32).
__global__ void f32_to_i32_kernel(float *D, int64_t ld, int64_t n, int64_t rows) {
  for (int64_t i = blockIdx.y; i < rows; i += gridDim.y)
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
      const float v = D[i * ld + j];
      reinterpret_cast<int32_t *>(D)[i * ld + j] = v < __int_as_float(0x7f800000) ? (int32_t)v : 0x3FFFFFFF;
    }
}

// Copy the `rows` x n result out of the padded workspace (unpad).
template <typename T>
__global__ void unpad_kernel(const T *D, int64_t ld, int64_t n, T *dst, int64_t ldd, int64_t rows) {
  for (int64_t i = blockIdx.y; i < rows; i += gridDim.y)
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x)
      dst[i * ldd + j] = D[i * ld + j];
}

// Host pipeline (fw_api.cu): a chunk's final distances into a dense output
// buffer (pitch ldo, n columns), out of place — the working rows stay intact because they
// are still read as pivot strips by the rounds other chunks have left. decode: keys ->
// distances; O = int32_t with T = float: FP32 compute back to INT32 storage (+inf -> FW_INF_I32).
template <typename O, typename T> __device__ __forceinline__ O to_storage(T v) { return (O)v; }
template <> __device__ __forceinline__ int32_t to_storage<int32_t, float>(float v) {
  return v < __int_as_float(0x7f800000) ? (int32_t)v : 0x3FFFFFFF;
}
template <typename T, typename O>
__global__ void emit_rows_kernel(const T *D, int64_t ld, int64_t n, int64_t rows, O *out, int64_t ldo,
                                 int decode) {
  for (int64_t i = blockIdx.y; i < rows; i += gridDim.y)
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
      const T v = D[i * ld + j];
      out[i * ldo + j] = to_storage<O, T>(decode ? Num<T>::decode(v) : v);
    }
}

// ---------------------------------------------------------------------------------
// TAG-mode post-pass, step 1 (reading R9): for each (i,j) whose last strict improvement
// happened in round K = tags[i][j] >= 0, find k* = the first k in block K, k not in {i,j},
// minimising D[i][k] + D[k][j] over the FINAL D. That minimum is D[i][j] in exact arithmetic:
// the improving k of round K reached D[i][j], later rounds only lowered D[i][k] and D[k][j],
// and the final D satisfies the triangle inequality; with rounding the arg-min is the most
// robust choice. k* is an intermediate vertex of a shortest i->j path, i.e. the paper's
// "most recently added intermediate node" form of P. Overwrites tags with k*.
//
// One CTA per row i (row i of D staged in shared memory when it fits); FOUR lanes per element
// (resolve_lastk_quad_kernel below); the kernel reads ~4*BS bytes of D^T per tagged element
// (~n^2 * 512 B at BS = 128).

// Dt = D^T in BLOCK PANELS: for every block K of BS rows, panel K is the n_pad x BS matrix
// Dt[(K n_pad + j) BS + k] = D[K BS + k][j] — so the column segment D[K BS .. K BS + BS)[j] the
// resolve searches is BS contiguous elements, and the panels of a block-row range are ONE
// contiguous range of Dt (a rank of a block-row partition transposes only its own rows and the
// ranks exchange their panel ranges, DESIGN.md §4.5 / §9). Rows [r0, r0 + rows) of D (global
// rows g0 + r0 ..), pitch ld; 32 x 32 shared-memory tiles. The diagonal (global row == column)
// is written as INF: the resolve below then never picks k = j (D[i][j] + D[j][j] = D[i][j]
// holds trivially) without testing for it. BS is a template parameter: the panel index and
// offset are shifts (with a run-time BS, the 64-bit divisions made the kernel issue-bound at
// 1.8 TB/s: 4.8 ms for the 8.6 GB of C5).
template <typename T, int BS>
__global__ void transpose_panels_kernel(const T *D, int64_t ld, int64_t rows, int64_t cols, int64_t g0, T *Dt) {
  __shared__ T tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t r = r0 + y, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[y][threadIdx.x] = D[r * ld + c];
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t c = c0 + y, r = r0 + threadIdx.x, gr = g0 + r;
    if (r < rows && c < cols)
      Dt[((gr / BS) * cols + c) * BS + gr % BS] = gr == c ? Num<T>::inf() : tile[threadIdx.x][y];
  }
}

// The search, FOUR lanes per element (8 elements per warp): lane q of element e takes the 16-B
// granules 4s' + q of block K (s' = s ^ (e & 1), s < BS/16), i.e. BS/4 candidates, and the quad
// takes the smallest of its four first hits with two shuffles. A warp spends ~16 instructions
// per element; the round-1/2 kernel with one warp per element spent ~60 and was ALU-issue bound
// (ncu at C2: 58.6 warp instructions per element, ALU pipe 69%, 1.42 ms; this kernel 0.86 ms). The four
// lanes of an element read 64 contiguous bytes of D^T per load (coalesced); the step swap for
// odd elements puts the 8 elements of a warp evenly on the two halves of the shared-memory bank
// space, so an LDS.128 of row i takes the minimum 4 wavefronts whatever the tags. The D^T loads
// of the next element are in flight while the current one is searched (two register stages).
template <typename T> __device__ __forceinline__ void add4(T (&o)[4], const typename Vec4<T>::V &a,
                                                             const typename Vec4<T>::V &b) {
  o[0] = a.x + b.x; o[1] = a.y + b.y; o[2] = a.z + b.z; o[3] = a.w + b.w;
}
template <> __device__ __forceinline__ void add4<float>(float (&o)[4], const float4 &a, const float4 &b) {
  const float2 lo = __fadd2_rn(make_float2(a.x, a.y), make_float2(b.x, b.y));   // FADD2: one rounded add each
  const float2 hi = __fadd2_rn(make_float2(a.z, a.w), make_float2(b.z, b.w));
  o[0] = lo.x; o[1] = lo.y; o[2] = hi.x; o[3] = hi.y;
}

template <typename T, int BS, bool SMEM>
__global__ void __launch_bounds__(512, 1)
resolve_lastk_quad_kernel(const T *D, const T *Dt, int64_t ld, int64_t ldt, int64_t row0, int64_t n,
                          int64_t n_pad, int32_t *tags) {
  constexpr int NS = BS / 16;              // 16-B granule steps per lane
  constexpr int kNone = 0x40000000;        // "no hit" (above every k, and k + 3 stays positive)
  using V = typename Vec4<T>::V;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *srow = reinterpret_cast<T *>(smem_raw);
  const int64_t li = blockIdx.x;
  const int gi = (int)(row0 + li), nn = (int)n;
  const T *Drow = D + li * ld;
  int32_t *trow = tags + li * ld;
  if constexpr (SMEM) {
    // row i with D[i][i] read as INF (k = i never picked); k = j is excluded by Dt's INF diagonal
    for (int j = threadIdx.x; j < (int)n_pad; j += blockDim.x) srow[j] = j == gi ? Num<T>::inf() : Drow[j];
    __syncthreads();
  }
  const T *A = SMEM ? srow : Drow;
  const int lane = threadIdx.x & 31, q = lane & 3, e = lane >> 2;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int step = nw * 8;
  const int sw = (e & 1) * 16;             // granule s of an odd element is s ^ 1: +16 (s even), -16 (s odd)
  const unsigned qmask = 0xfu << (lane & ~3);
  auto load = [&](int j, int t, V (&b)[NS]) {
    const T *bp = Dt + ((int64_t)max(t, 0) * ldt + min(j, nn - 1)) * BS + 4 * q;   // panel t, row j
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (t >= 0) b[s] = *reinterpret_cast<const V *>(bp + 16 * s + ((s & 1) ? -sw : sw));
  };
  auto search = [&](int j, int t, const V (&b)[NS]) {
    if (t < 0) return;
    // reading R9: k* = the FIRST k of block K, k not in {i, j}, with D[i][k] + D[k][j] <= D[i][j]
    const T dij = A[j];
    const int kq = t * BS + 4 * q;
    int kl = kNone;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int k0 = kq + 16 * s + ((s & 1) ? -sw : sw);
      const V a = *reinterpret_cast<const V *>(A + k0);
      T sum[4];
      add4<T>(sum, a, b[s]);
      int kf = kNone;                      // first hit among the granule's 4 candidates
#pragma unroll
      for (int c = 3; c >= 0; --c) kf = (sum[c] <= dij && (SMEM || k0 + c != gi)) ? c : kf;
      kl = min(kl, k0 + kf);
    }
    kl = min(kl, __shfl_xor_sync(qmask, kl, 1));
    kl = min(kl, __shfl_xor_sync(qmask, kl, 2));
    if (q == 0) trow[j] = kl >= kNone ? -1 : kl;
  };
  // pipeline: element m's D^T segment is in registers (ba / bb alternate) while m + 1's loads are
  // in flight, and the tags run two elements further ahead, so no D^T load waits on its tag
  auto tag_of = [&](int j) { return j < nn ? trow[j] : -1; };
  V ba[NS], bb[NS];
  int j0 = warp * 8 + e;
  int ta = tag_of(j0), tb = tag_of(j0 + step), tc = tag_of(j0 + 2 * step), td = tag_of(j0 + 3 * step);
  load(j0, ta, ba);
  for (; j0 - e < nn; j0 += 2 * step) {
    const int t4 = tag_of(j0 + 4 * step), t5 = tag_of(j0 + 5 * step);
    load(j0 + step, tb, bb);
    search(j0, ta, ba);
    if (j0 + step - e >= nn) break;
    load(j0 + 2 * step, tc, ba);
    search(j0 + step, tb, bb);
    ta = tc;
    tb = td;
    tc = t4;
    td = t5;
  }
}

// TAG-mode post-pass, step 2 (NEXT-HOP mode, readings R1/R10): per row i, next[i][j] = j if
// (i,j) was never improved (direct edge), else next[i][k*] (k* = LAST_K[i][j]); resolved by
// pointer jumping on row i in shared memory (or in place when the row does not fit). With
// positive weights D[i][k*] < D[i][j], so chains are acyclic. Then the sentinels:
// next[i][i] = i, next[i][j] = -1 when D[i][j] is INF. LAST_K mode only applies the
// sentinels (diagonal and unreachable -> -1). flags bit 3: a chain did not converge.
// decode = 1 (keyed mode): also turns the row's keys into distances (Num<T>::decode).
template <typename T>
__global__ void __launch_bounds__(1024)
finalize_paths_kernel(T *D, int32_t *P, int64_t ld, int64_t row0, int64_t n, int next_hop,
                      int use_smem, int *flags, int decode) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t li = blockIdx.x;          // local row
  const int64_t i = row0 + li;            // global row
  int32_t *row = P + li * ld;
  T *Drow = D + li * ld;
  if (!next_hop) {
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
      const T d = Drow[j];
      if (decode) Drow[j] = Num<T>::decode(d);
      if (j == i || !Num<T>::finite(d)) row[j] = -1;
    }
    return;
  }
  int32_t *v = use_smem ? reinterpret_cast<int32_t *>(smem_raw) : row;
  // 16-B vectors for the row passes when rows are 16-B aligned (ld, n multiples of 4)
  const bool vec = (n % 4 == 0) && (ld % 4 == 0);
  const int64_t j0 = vec ? n : 0;     // scalar loops start here (all of the row when !vec)
  if (vec) {
    for (int64_t q = threadIdx.x; q < n / 4; q += blockDim.x) {
      const int4 t = reinterpret_cast<const int4 *>(row)[q];
      const int32_t j = (int32_t)(4 * q);
      reinterpret_cast<int4 *>(v)[q] = make_int4(t.x < 0 ? (j | kTerm) : t.x, t.y < 0 ? ((j + 1) | kTerm) : t.y,
                                                 t.z < 0 ? ((j + 2) | kTerm) : t.z, t.w < 0 ? ((j + 3) | kTerm) : t.w);
    }
  }
  for (int64_t j = j0 + threadIdx.x; j < n; j += blockDim.x) {
    const int32_t t = row[j];
    v[j] = t < 0 ? (int32_t)(j | kTerm) : t;
  }
  __syncthreads();
  int sweeps = 0;
  for (;;) {
    int active = 0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
      const int32_t x = v[j];
      if (!(x & kTerm)) {
        const int32_t y = ((volatile int32_t *)v)[x];
        v[j] = y;
        active |= !(y & kTerm);
      }
    }
    active = __syncthreads_or(active);
    if (!active) break;
    if (++sweeps > 64) {
      if (threadIdx.x == 0) atomicOr(flags, 8);
      break;
    }
  }
  auto final_next = [&](int32_t x, T d, int64_t j) -> int32_t {
    int32_t out = (x & kTerm) ? (x & ~kTerm) : -1;
    if (j == i) out = (int32_t)i;
    else if (!Num<T>::finite(d)) out = -1;
    return out;
  };
  if (vec) {
    using VT = typename Vec4<T>::V;
    for (int64_t q = threadIdx.x; q < n / 4; q += blockDim.x) {
      const int4 x = reinterpret_cast<const int4 *>(v)[q];
      const VT d = reinterpret_cast<const VT *>(Drow)[q];
      if (decode) {
        VT o;
        o.x = Num<T>::decode(d.x); o.y = Num<T>::decode(d.y); o.z = Num<T>::decode(d.z); o.w = Num<T>::decode(d.w);
        reinterpret_cast<VT *>(Drow)[q] = o;
      }
      const int64_t j = 4 * q;
      reinterpret_cast<int4 *>(row)[q] = make_int4(final_next(x.x, d.x, j), final_next(x.y, d.y, j + 1),
                                                   final_next(x.z, d.z, j + 2), final_next(x.w, d.w, j + 3));
    }
  }
  for (int64_t j = j0 + threadIdx.x; j < n; j += blockDim.x) {
    const int32_t x = v[j];
    const T d = Drow[j];
    if (decode) Drow[j] = Num<T>::decode(d);
    row[j] = final_next(x, d, j);
  }
}

}  // namespace fwb

// fw_kernels.cuh — sm_100a kernels of the blocked Floyd–Warshall hot path.
//
// Method: arxiv 1811.01201 §4.1. One round K relaxes every pair
// through the BS intermediate vertices k in [kb, kb+BS), kb = K*BS, in three phases:
//   phase 1     diagonal block D_KK, self-dependent: sequential k-loop in smem
//   phase 2 pivot row strip D_KJ and column strip D_IK, each relaxed through
//                        the closed D_KK* as a min-plus product (reading R7)
//   phase 3     every other block D_IJ <- min(D_IJ, D_IK (x) D_KJ)
// The loop body of the paper's FW_BLOCK ("one addition, one comparison") becomes
// the relaxation microkernel below: FP32 uses packed FADD2 (2 adds per instruction) +
// 3-input FMNMX3 (2 mins per instruction), i.e. one issue slot per relaxation;
// INT32 uses VIADDMNMX (fused add+min). The P update is taken off the per-relaxation
// path (reading R9): the epilogue writes the round number K as a tag for every element
// whose distance strictly improved; a post-pass resolves tags into P.
//
// Layout: D and the tag/P matrix are row-major,
// n_pad x n_pad, leading dimension ld (a multiple of 128 elements here).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

namespace fwb {

constexpr int kThreads = 256;          // tile kernel: 16 x 16 threads
constexpr int kTag = 0x40000000;       // terminal bit used by the next-hop pointer jumping

template <typename T> struct Num;
template <> struct Num<float> {
  static constexpr bool kIsInt = false;
  static __device__ __forceinline__ float inf() { return __int_as_float(0x7f800000); }
  static __device__ __forceinline__ bool bad(float v) { return !(v >= 0.0f); }  // NaN or < 0
  static __device__ __forceinline__ bool finite(float v) { return v < inf(); }
};
template <> struct Num<int32_t> {
  static constexpr bool kIsInt = true;
  static __device__ __forceinline__ int32_t inf() { return 0x3FFFFFFF; }
  static __device__ __forceinline__ bool bad(int32_t v) { return v < 0 || v > 0x3FFFFFFF; }
  static __device__ __forceinline__ bool finite(int32_t v) { return v < 0x3FFFFFFF; }
};

// ---------------------------------------------------------------------------------
// cp.async helpers (LDGSTS): global -> shared without staging registers.
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------------
// Relaxation microkernel: acc = min(acc, a.x+b.x, a.y+b.y, a.z+b.z, a.w+b.w)
// where a = (a_ik, a_ik+1, a_ik+2, a_ik+3) and b = (b_kj, b_k+1j, b_k+2j, b_k+3j):
// four relaxations of one (i,j) pair through four consecutive k (P:125 loop body).
// Every sum is a single IEEE round-to-nearest add; min is exact, so the order in
// which the four candidates are folded does not change the result (reading R8).
template <typename T> struct Relax;
template <> struct Relax<float> {
  using V = float4;
  static __device__ __forceinline__ void run(float &acc, const float4 &a, const float4 &b) {
    const float2 s01 = __fadd2_rn(make_float2(a.x, a.y), make_float2(b.x, b.y));  // FADD2
    const float2 s23 = __fadd2_rn(make_float2(a.z, a.w), make_float2(b.z, b.w));  // FADD2
    acc = fminf(acc, fminf(s01.x, s01.y));                                          // FMNMX3
    acc = fminf(acc, fminf(s23.x, s23.y));                                          // FMNMX3
  }
};
template <> struct Relax<int32_t> {
  using V = int4;
  static __device__ __forceinline__ void run(int32_t &acc, const int4 &a, const int4 &b) {
    acc = __viaddmin_s32(a.x, b.x, acc);   // VIADDMNMX: min(a+b, acc)
    acc = __viaddmin_s32(a.y, b.y, acc);
    acc = __viaddmin_s32(a.z, b.z, acc);
    acc = __viaddmin_s32(a.w, b.w, acc);
  }
};

template <int TM, int TN, int BK>
struct TileSmem {
  static constexpr int kAStride = BK + 4;             // padded A row (16 B pad: no bank conflicts)
  static constexpr int kA = TM * kAStride;            // elements per A stage
  static constexpr int kB = BK * TN;                  // elements per B stage (k-quad interleaved)
  static constexpr int kStage = kA + kB;
  static constexpr int kBytes = 2 * kStage * 4;       // two stages (double buffering)
};

// ---------------------------------------------------------------------------------
// Min-plus tile kernel used by phases 2 and 3:
//   C[i][j] <- min(C[i][j], min_{k<Kd} A[i][k] + B[k][j])   for the tile's (i,j)
// excluding rows in [mr_lo, mr_hi) and columns in [mc_lo, mc_hi) (those belong to
// the strips phase 2 owns). If TAGS, every element whose value strictly
// decreased gets tags[i][j] = tag (the round number K; reading R9).
// A is TM x Kd (row-major, lda), B is Kd x TN (row-major, ldb). The CTA tile is TM x TN,
// each of the 256 threads owns (TM/16) x (TN/16) elements strided by 16 in i and j.
// The k dimension is streamed in chunks of BK through two shared-memory stages with
// cp.async. A is staged row-major [i][k] (16-B copies), B k-quad interleaved
// [k/4][j][k%4] (4-B copies) so one LDS.128 yields b_kj..b_k+3,j for FADD2 pairs.
// In-place use (phase 2: C aliases A or B) is safe: a CTA reads all of its A/B chunks
// before its epilogue writes, and no other CTA writes the region it reads.
template <typename T, int TM, int TN, int BK, bool TAGS>
__global__ void __launch_bounds__(kThreads, 2)
minplus_tile_kernel(T *C, int64_t ldc, const T *A, int64_t lda, const T *B, int64_t ldb,
                    int32_t *tags, int64_t ldt, int Kd, int mr_lo, int mr_hi, int mc_lo,
                    int mc_hi, int tag) {
  using S = TileSmem<TM, TN, BK>;
  using V = typename Relax<T>::V;
  constexpr int RM = TM / 16, RN = TN / 16;
  static_assert(BK % 4 == 0 && TM % 16 == 0 && TN % 16 == 0, "tile shape");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *smem = reinterpret_cast<T *>(smem_raw);

  const int i0 = blockIdx.y * TM, j0 = blockIdx.x * TN;
  // whole tile inside an excluded strip: nothing to do
  if ((i0 >= mr_lo && i0 + TM <= mr_hi) || (j0 >= mc_lo && j0 + TN <= mc_hi)) return;

  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  // Per-thread copy assignments (fixed across chunks; only the k offset advances).
  // A: float4 number idx = tid + 256*t covers row r = idx / (BK/4), column quad idx % (BK/4).
  constexpr int AQ = BK / 4;                          // float4 per A row chunk
  constexpr int A_ITERS = (TM * AQ + kThreads - 1) / kThreads;
  constexpr int A_ROWS_PER_ITER = kThreads / AQ;
  static_assert(kThreads % AQ == 0, "A copy mapping");
  const int a_r = tid / AQ, a_c = (tid % AQ) * 4;
  const T *a_src = A + (int64_t)(i0 + a_r) * lda + a_c;
  const int a_dst = a_r * S::kAStride + a_c;
  // B: element idx = tid + 256*t covers row k = idx / TN, column j = idx % TN.
  constexpr int B_ITERS = BK * TN / kThreads;
  constexpr int B_ROWS_PER_ITER = kThreads / TN;
  static_assert(kThreads % TN == 0 && (BK * TN) % kThreads == 0, "B copy mapping");
  const int b_k = tid / TN, b_j = tid % TN;
  const T *b_src = B + (int64_t)b_k * ldb + j0 + b_j;

  auto load_chunk = [&](int stage, int k0) {
    T *as = smem + stage * S::kStage;
    T *bs = as + S::kA;
    const T *ap = a_src + k0;
#pragma unroll
    for (int t = 0; t < A_ITERS; ++t) {
      if (A_ITERS * kThreads == TM * AQ || a_r + t * A_ROWS_PER_ITER < TM)
        cp_async16(as + a_dst + t * A_ROWS_PER_ITER * S::kAStride, ap + (int64_t)t * A_ROWS_PER_ITER * lda);
    }
    const T *bp = b_src + (int64_t)k0 * ldb;
#pragma unroll
    for (int t = 0; t < B_ITERS; ++t) {
      const int k = b_k + t * B_ROWS_PER_ITER;
      cp_async4(bs + ((k >> 2) * TN + b_j) * 4 + (k & 3), bp + (int64_t)t * B_ROWS_PER_ITER * ldb);
    }
    cp_async_commit();
  };

  T acc[RM][RN];
#pragma unroll
  for (int r = 0; r < RM; ++r)
#pragma unroll
    for (int c = 0; c < RN; ++c) acc[r][c] = Num<T>::inf();

  const int nch = Kd / BK;
  load_chunk(0, 0);
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) {
      load_chunk((ch + 1) & 1, (ch + 1) * BK);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const T *as = smem + (ch & 1) * S::kStage + ty * S::kAStride;
    const T *bs = smem + (ch & 1) * S::kStage + S::kA + tx * 4;
#pragma unroll
    for (int q = 0; q < BK / 4; ++q) {
      V b[RN];
#pragma unroll
      for (int c = 0; c < RN; ++c) b[c] = *reinterpret_cast<const V *>(bs + (q * TN + 16 * c) * 4);
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        const V a = *reinterpret_cast<const V *>(as + 16 * r * S::kAStride + 4 * q);
#pragma unroll
        for (int c = 0; c < RN; ++c) Relax<T>::run(acc[r][c], a, b[c]);
      }
    }
    __syncthreads();
  }

  // Epilogue: compare with the current value, store strict improvements (+ tag K).
#pragma unroll
  for (int r = 0; r < RM; ++r) {
    const int i = i0 + ty + 16 * r;
    const bool row_ok = !(i >= mr_lo && i < mr_hi);
    T old[RN];
#pragma unroll
    for (int c = 0; c < RN; ++c) old[c] = C[(int64_t)i * ldc + j0 + tx + 16 * c];
#pragma unroll
    for (int c = 0; c < RN; ++c) {
      const int j = j0 + tx + 16 * c;
      const bool ok = row_ok && !(j >= mc_lo && j < mc_hi);
      if (ok && acc[r][c] < old[c]) {
        C[(int64_t)i * ldc + j] = acc[r][c];
        if (TAGS) tags[(int64_t)i * ldt + j] = tag;
      }
    }
  }
}

// ---------------------------------------------------------------------------------
// Phase 1: closure of the diagonal block D_KK in shared memory. For each k in
// the block (in order), d[a][b] = min(d[a][b], d[a][k] + d[k][b]) (strict '<'). Row k and
// column k are invariant during step k because d[k][k] = 0, so updating in place with
// one barrier per k is exact. Elements that strictly improved get tag K.
template <typename T, bool TAGS>
__global__ void __launch_bounds__(1024)
phase1_kernel(T *D, int64_t ld, int32_t *tags, int64_t ldt, int kb, int BS, int tag) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *s = reinterpret_cast<T *>(smem_raw);
  const int nel = BS * BS;
  T *Dk = D + (int64_t)kb * ld + kb;
  for (int e = threadIdx.x; e < nel; e += blockDim.x) s[e] = Dk[(int64_t)(e / BS) * ld + e % BS];
  __syncthreads();
  for (int k = 0; k < BS; ++k) {
    for (int e = threadIdx.x; e < nel; e += blockDim.x) {
      const int a = e / BS, b = e - a * BS;
      const T v = s[a * BS + k] + s[k * BS + b];
      if (v < s[e]) s[e] = v;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < nel; e += blockDim.x) {
    const int64_t off = (int64_t)(e / BS) * ld + e % BS;
    if (s[e] < Dk[off]) {
      Dk[off] = s[e];
      if (TAGS) tags[(int64_t)(kb + e / BS) * ldt + kb + e % BS] = tag;
    }
  }
}

// ---------------------------------------------------------------------------------
// Validation (read-only, before anything is written: fw.h error contract).
// flags bit 0: out-of-domain value. maxw: max finite off-diagonal weight (INT32 only).
template <typename T>
__global__ void validate_kernel(const T *src, int64_t lds, int64_t n, int *flags, int *maxw) {
  int bad = 0, mx = 0;
  const int64_t total = n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    const T v = src[i * lds + j];
    if (i == j) continue;  // the diagonal is overwritten with 0 (R4)
    if (Num<T>::bad(v)) bad = 1;
    if (Num<T>::kIsInt && !Num<T>::bad(v) && Num<T>::finite(v)) {
      const int iv = (int)v;
      mx = iv > mx ? iv : mx;
    }
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) {
    if (bad) atomicOr(flags, 1);
    atomicMax(maxw, mx);
  }
}

// Copy W (n x n, lds) into the padded n_pad x n_pad workspace (ld): padded entries INF,
// diagonal 0 (R4, R11); tags/P initialised to -1 ("no improvement yet"). src may alias D
// (in-place solve) — each element is read then written by the same thread.
template <typename T>
__global__ void init_kernel(const T *src, int64_t lds, int64_t n, T *D, int64_t ld, int64_t n_pad,
                            int32_t *tags, int64_t ldt) {
  const int64_t i = blockIdx.y;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_pad;
       j += (int64_t)gridDim.x * blockDim.x) {
    T v = (i < n && j < n) ? src[i * lds + j] : Num<T>::inf();
    if (i == j) v = 0;
    D[i * ld + j] = v;
    if (tags) tags[i * ldt + j] = -1;
  }
}

// Copy the n x n result out of the padded workspace (unpad).
template <typename T>
__global__ void unpad_kernel(const T *D, int64_t ld, int64_t n, T *dst, int64_t ldd) {
  const int64_t i = blockIdx.y;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    dst[i * ldd + j] = D[i * ld + j];
}

// ---------------------------------------------------------------------------------
// Post-pass step 1 (reading R9): for each (i,j) whose last strict improvement happened in
// round K = tags[i][j] >= 0, find k* = the first k in block K, k not in {i,j}, minimising
// D[i][k] + D[k][j] over the FINAL D. In exact arithmetic D[i][k*] + D[k*][j] = D[i][j]
// (the improving k of round K attains it and final D obeys the triangle inequality), so
// k* is a "most recently added intermediate node" in the paper's sense.
// Overwrites tags in place with k* (LAST_K form); untagged entries stay -1.
template <typename T>
__global__ void resolve_lastk_kernel(const T *D, int64_t ld, int32_t *tags, int64_t ldt,
                                     int64_t n, int BS) {
  const int64_t i = blockIdx.y;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int t = tags[i * ldt + j];
  if (t < 0) return;
  const int64_t kb = (int64_t)t * BS;
  const int64_t ke = kb + BS < n ? kb + BS : n;
  T best = Num<T>::inf();
  int ks = -1;
  const T *Di = D + i * ld;
  for (int64_t k = kb; k < ke; ++k) {
    if (k == i || k == j) continue;
    const T s = Di[k] + D[k * ld + j];
    if (s < best) { best = s; ks = (int)k; }
  }
  tags[i * ldt + j] = ks;
}

// Post-pass step 2 (NEXT-HOP mode, reading R1/R10): per row i, next[i][j] = j if (i,j) was
// never improved (direct edge), else next[i][k*] (k* = LAST_K[i][j]); resolved by pointer
// jumping on row i in shared memory (or in place in global memory when the row does not
// fit). With positive weights D[i][k*] < D[i][j], so chains are acyclic. Then the
// sentinels: next[i][i] = i, next[i][j] = -1 when D[i][j] is INF. LAST_K mode only applies
// the sentinels (diagonal and unreachable -> -1). flags bit 1: chain did not converge.
template <typename T>
__global__ void __launch_bounds__(1024)
finalize_paths_kernel(const T *D, int64_t ld, int32_t *P, int64_t ldp, int64_t n, int next_hop,
                      int use_smem, int *flags) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t i = blockIdx.x;
  int32_t *row = P + i * ldp;
  const T *Drow = D + i * ld;
  if (!next_hop) {
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x)
      if (j == i || !Num<T>::finite(Drow[j])) row[j] = -1;
    return;
  }
  int32_t *v = use_smem ? reinterpret_cast<int32_t *>(smem_raw) : row;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    const int32_t t = row[j];
    v[j] = t < 0 ? (int32_t)(j | kTag) : t;
  }
  __syncthreads();
  int sweeps = 0;
  for (;;) {
    int active = 0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
      const int32_t x = v[j];
      if (!(x & kTag)) {
        const int32_t y = ((volatile int32_t *)v)[x];
        v[j] = y;
        active |= !(y & kTag);
      }
    }
    active = __syncthreads_or(active);
    if (!active) break;
    if (++sweeps > 64) {
      if (threadIdx.x == 0) atomicOr(flags, 2);
      break;
    }
  }
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    const int32_t x = v[j];
    int32_t out = (x & kTag) ? (x & ~kTag) : -1;
    if (j == i) out = (int32_t)i;
    else if (!Num<T>::finite(Drow[j])) out = -1;
    row[j] = out;
  }
}

}  // namespace fwb

// fw_api.cu — C ABI (include/fw.h) and the single-GPU round driver of the blocked
// Floyd–Warshall solve (arxiv 1811.01201 §4.1).
//
// Round loop (OpenMP structure of P:151-155 mapped to stream-ordered
// launches): for K in 0..R-1: phase 1 on D_KK (1 CTA), phase 2 on the pivot row strip
// and column strip (two launches), phase 3 on the rest (one launch of 128x128 tiles).
// Stream order replaces the paper's implicit OpenMP barriers; the host only enqueues.
// After the rounds, the post-pass turns the round tags into P (reading R9).
#include "fw_kernels.cuh"
#include "../../include/fw.h"

#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <type_traits>
#include <vector>

using namespace fwb;

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(FW_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),    \
                  __FILE__, __LINE__);                                                 \
  } while (0)

#define TRY(call)                 \
  do {                            \
    int rc_ = (call);             \
    if (rc_ != FW_OK) return rc_; \
  } while (0)

struct DevBuf {
  void *p = nullptr;
  size_t bytes = 0;
  int ensure(size_t want) {
    if (bytes >= want) return FW_OK;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    if (cudaMalloc(&p, want) != cudaSuccess) {
      cudaGetLastError();
      return fail(FW_ENOMEM, "cudaMalloc(%zu) failed", want);
    }
    bytes = want;
    return FW_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

struct Ctx {
  int dev = 0;
  unsigned flags = 0;
  cudaStream_t stream = nullptr;   // internal stream for the host entry points
  DevBuf ws_d, ws_t;               // padded workspaces (D, tags/P)
  DevBuf user_d, user_t;           // device copies of host buffers (host entry points)
  DevBuf scratch;                  // validation flags
  void *pinned = nullptr;          // staging for pageable host buffers
  size_t pinned_bytes = 0;
  std::vector<cudaEvent_t> events;
  fw_stats stats{};
  bool has_stats = false;
};

Ctx *g_ctx = nullptr;

constexpr int kBK = 32;
constexpr size_t kStageBytes = 64ull << 20;  // pinned staging chunk

int ensure_events(Ctx &c, size_t count) {
  while (c.events.size() < count) {
    cudaEvent_t e;
    CU(cudaEventCreate(&e));
    c.events.push_back(e);
  }
  return FW_OK;
}

// ---- kernel launch wrappers ---------------------------------------------------------
template <typename T, int TM, int TN, bool TAGS>
int launch_tile(dim3 grid, cudaStream_t st, T *C, int64_t ldc, const T *A, int64_t lda,
                const T *B, int64_t ldb, int32_t *tags, int64_t ldt, int Kd, int mr_lo,
                int mr_hi, int mc_lo, int mc_hi, int tag) {
  constexpr int bytes = TileSmem<TM, TN, kBK>::kBytes;
  auto kern = minplus_tile_kernel<T, TM, TN, kBK, TAGS>;
  static bool configured = false;  // per instantiation
  if (!configured) {
    CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    configured = true;
  }
  kern<<<grid, kThreads, bytes, st>>>(C, ldc, A, lda, B, ldb, tags, ldt, Kd, mr_lo, mr_hi,
                                      mc_lo, mc_hi, tag);
  CU(cudaGetLastError());
  return FW_OK;
}

template <typename T, bool TAGS>
int launch_phase1(cudaStream_t st, T *D, int64_t ld, int32_t *tags, int kb, int BS, int K) {
  const int bytes = BS * BS * (int)sizeof(T);
  auto kern = phase1_kernel<T, TAGS>;
  static bool configured = false;
  if (!configured) {
    CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 128 * 4));
    configured = true;
  }
  kern<<<1, 1024, bytes, st>>>(D, ld, tags, ld, kb, BS, K);
  CU(cudaGetLastError());
  return FW_OK;
}

// Phase 2: row strip D[kb:kb+BS, :] and column strip D[:, kb:kb+BS] relaxed
// through the closed diagonal block D_KK* (min-plus product form, reading R7).
template <typename T, bool TAGS, int BS>
int launch_phase2_bs(cudaStream_t st, T *D, int64_t ld, int32_t *tags, int64_t n_pad, int kb,
                     int K) {
  T *rowC = D + (int64_t)kb * ld;
  T *colC = D + kb;
  const T *Dkk = D + (int64_t)kb * ld + kb;
  int32_t *rowT = tags ? tags + (int64_t)kb * ld : nullptr;
  int32_t *colT = tags ? tags + kb : nullptr;
  const int tiles = (int)(n_pad / 128);
  // row strip: C = A? no: C = B (in place), A = D_KK*; exclude the diagonal block columns
  TRY((launch_tile<T, BS, 128, TAGS>(dim3(tiles, 1), st, rowC, ld, Dkk, ld, rowC, ld, rowT, ld,
                                     BS, 0, 0, kb, kb + BS, K)));
  // column strip: C = A (in place), B = D_KK*; exclude the diagonal block rows
  TRY((launch_tile<T, 128, BS, TAGS>(dim3(1, tiles), st, colC, ld, colC, ld, Dkk, ld, colT, ld,
                                     BS, kb, kb + BS, 0, 0, K)));
  return FW_OK;
}

template <typename T, bool TAGS>
int launch_phase2(cudaStream_t st, T *D, int64_t ld, int32_t *tags, int64_t n_pad, int kb,
                  int BS, int K) {
  switch (BS) {
    case 32: return launch_phase2_bs<T, TAGS, 32>(st, D, ld, tags, n_pad, kb, K);
    case 64: return launch_phase2_bs<T, TAGS, 64>(st, D, ld, tags, n_pad, kb, K);
    case 128: return launch_phase2_bs<T, TAGS, 128>(st, D, ld, tags, n_pad, kb, K);
  }
  return fail(FW_EINVAL, "unsupported block size %d", BS);
}

// Phase 3: D_IJ <- min(D_IJ, D_IK (x) D_KJ) for all I != K, J != K.
template <typename T, bool TAGS>
int launch_phase3(cudaStream_t st, T *D, int64_t ld, int32_t *tags, int64_t n_pad, int kb,
                  int BS, int K) {
  const int tiles = (int)(n_pad / 128);
  return launch_tile<T, 128, 128, TAGS>(dim3(tiles, tiles), st, D, ld, D + kb, ld,
                                        D + (int64_t)kb * ld, ld, tags, ld, BS, kb, kb + BS, kb,
                                        kb + BS, K);
}

template <typename T>
constexpr bool is_int_v() { return std::is_integral<T>::value; }

// ---- the solve on device buffers ----------------------------------------------------
// src: n rows of ld_src elements (in/out); next: n rows of ld_next int32 or nullptr.
template <typename T>
int solve_device(Ctx &c, T *src, int64_t ld_src, int32_t *next, int64_t ld_next, int64_t n,
                 int BS, cudaStream_t st) {
  const bool int_t = is_int_v<T>();
  const int64_t n_pad = (n + 127) / 128 * 128;
  const bool want_p = next != nullptr;
  const int path_mode = want_p ? ((c.flags & FW_PATH_LAST_K) ? 1 : 0) : -1;
  const bool timing = (c.flags & FW_TIMING) != 0;

  // 1. validation (read-only; outputs untouched on error)
  TRY(c.scratch.ensure(64));
  int *d_flags = static_cast<int *>(c.scratch.p);
  CU(cudaMemsetAsync(d_flags, 0, 16, st));
  {
    const int64_t total = n * n;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    validate_kernel<T><<<std::max(blocks, 1), 256, 0, st>>>(src, ld_src, n, d_flags, d_flags + 1);
    CU(cudaGetLastError());
  }
  int h_flags[2] = {0, 0};
  CU(cudaMemcpyAsync(h_flags, d_flags, sizeof h_flags, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (h_flags[0] & 1)
    return fail(FW_EINVAL, int_t ? "weight outside [0, FW_INF_I32]" : "negative or NaN weight");
  if (int_t && n > 1 && (int64_t)(n - 1) * (int64_t)h_flags[1] >= (int64_t)FW_INF_I32)
    return fail(FW_ERANGE, "(n-1)*max_weight = %lld >= FW_INF_I32: finite path sums could reach INF",
                (long long)(n - 1) * h_flags[1]);

  // 2. placement: in place when the caller's buffer already has the padded layout
  const bool inplace = n == n_pad && ld_src == n && ((uintptr_t)src % 16 == 0) &&
                       (!want_p || (ld_next == n && (uintptr_t)next % 16 == 0));
  T *D = src;
  int32_t *Tg = next;
  int64_t ld = n;
  if (!inplace) {
    TRY(c.ws_d.ensure((size_t)n_pad * n_pad * sizeof(T)));
    D = static_cast<T *>(c.ws_d.p);
    if (want_p) {
      TRY(c.ws_t.ensure((size_t)n_pad * n_pad * sizeof(int32_t)));
      Tg = static_cast<int32_t *>(c.ws_t.p);
    }
    ld = n_pad;
  }

  const int R = (int)((n + BS - 1) / BS);  // rounds wholly inside the padding are skipped
  TRY(ensure_events(c, 4 + (timing ? 3 * (size_t)R + 2 : 0)));
  cudaEvent_t e_begin = c.events[0], e_end = c.events[1];
  CU(cudaEventRecord(e_begin, st));

  // 3. init: pad, diag 0, tags -1
  {
    dim3 g((unsigned)std::min<int64_t>((n_pad + 255) / 256, 64), (unsigned)n_pad);
    init_kernel<T><<<g, 256, 0, st>>>(src, ld_src, n, D, ld, n_pad, want_p ? Tg : nullptr, ld);
    CU(cudaGetLastError());
  }
  if (timing) CU(cudaEventRecord(c.events[3 + 3 * R], st));

  // 4. rounds
  for (int K = 0; K < R; ++K) {
    const int kb = K * BS;
    if (want_p) {
      TRY((launch_phase1<T, true>(st, D, ld, Tg, kb, BS, K)));
      if (timing) CU(cudaEventRecord(c.events[2 + 3 * K], st));
      TRY((launch_phase2<T, true>(st, D, ld, Tg, n_pad, kb, BS, K)));
      if (timing) CU(cudaEventRecord(c.events[3 + 3 * K], st));
      TRY((launch_phase3<T, true>(st, D, ld, Tg, n_pad, kb, BS, K)));
    } else {
      TRY((launch_phase1<T, false>(st, D, ld, nullptr, kb, BS, K)));
      if (timing) CU(cudaEventRecord(c.events[2 + 3 * K], st));
      TRY((launch_phase2<T, false>(st, D, ld, nullptr, n_pad, kb, BS, K)));
      if (timing) CU(cudaEventRecord(c.events[3 + 3 * K], st));
      TRY((launch_phase3<T, false>(st, D, ld, nullptr, n_pad, kb, BS, K)));
    }
    if (timing) CU(cudaEventRecord(c.events[4 + 3 * K], st));
  }

  // 5. post-pass: tags -> LAST_K -> next hop (reading R9/R10)
  if (want_p) {
    dim3 g((unsigned)((n + 255) / 256), (unsigned)n);
    resolve_lastk_kernel<T><<<g, 256, 0, st>>>(D, ld, Tg, ld, n, BS);
    CU(cudaGetLastError());
    const size_t row_bytes = (size_t)n * sizeof(int32_t);
    const int use_smem = row_bytes <= 200 * 1024;
    static bool configured = false;
    if (!configured) {
      CU(cudaFuncSetAttribute(finalize_paths_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              200 * 1024));
      configured = true;
    }
    finalize_paths_kernel<T><<<(unsigned)n, 1024, use_smem ? row_bytes : 0, st>>>(
        D, ld, Tg, ld, n, path_mode == 0, use_smem, d_flags);
    CU(cudaGetLastError());
  }
  if (timing) CU(cudaEventRecord(c.events[2 + 3 * R], st));

  // 6. unpad into the caller's buffers
  if (!inplace) {
    dim3 g((unsigned)std::min<int64_t>((n + 255) / 256, 64), (unsigned)n);
    unpad_kernel<T><<<g, 256, 0, st>>>(D, ld, n, src, ld_src);
    CU(cudaGetLastError());
    if (want_p) {
      unpad_kernel<int32_t><<<g, 256, 0, st>>>(Tg, ld, n, next, ld_next);
      CU(cudaGetLastError());
    }
  }
  CU(cudaEventRecord(e_end, st));
  CU(cudaMemcpyAsync(h_flags, d_flags, sizeof h_flags, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (h_flags[0] & 2)
    return fail(FW_ERANGE, "next-hop resolution did not converge (zero-weight cycle?)");

  fw_stats s{};
  s.n = n;
  s.n_pad = n_pad;
  s.block = BS;
  s.rounds = R;
  s.is_int = int_t;
  s.path_mode = path_mode;
  float ms = 0.f;
  CU(cudaEventElapsedTime(&ms, e_begin, e_end));
  s.solve_ms = ms;
  const double tiles_off = (double)(n_pad - BS);
  s.phase3_launches = R;
  s.phase3_relaxations = (double)R * tiles_off * tiles_off * BS;
  if (timing) {
    for (int K = 0; K < R; ++K) {
      float a = 0, b = 0, d = 0;
      CU(cudaEventElapsedTime(&a, K == 0 ? c.events[3 + 3 * R] : c.events[4 + 3 * (K - 1)], c.events[2 + 3 * K]));
      CU(cudaEventElapsedTime(&b, c.events[2 + 3 * K], c.events[3 + 3 * K]));
      CU(cudaEventElapsedTime(&d, c.events[3 + 3 * K], c.events[4 + 3 * K]));
      s.phase1_ms += a;
      s.phase2_ms += b;
      s.phase3_ms += d;
    }
    float p = 0;
    CU(cudaEventElapsedTime(&p, c.events[4 + 3 * (R - 1)], c.events[2 + 3 * R]));
    s.post_ms = p;
  }
  c.stats = s;
  c.has_stats = true;
  return FW_OK;
}

int pick_block(int64_t n, int block, int *BS) {
  if (block == 0) block = n >= 4096 ? 128 : 64;
  if (block != 32 && block != 64 && block != 128)
    return fail(FW_EINVAL, "block must be 0, 32, 64 or 128 (got %d)", block);
  *BS = block;
  return FW_OK;
}

int check_common(int64_t n, const void *dist, int block, int *BS) {
  if (!g_ctx) return fail(FW_ESTATE, "fw_init has not been called");
  if (n <= 0 || n > 65536) return fail(FW_EINVAL, "n must be in [1, 65536] (got %lld)", (long long)n);
  if (!dist) return fail(FW_EINVAL, "dist is NULL");
  return pick_block(n, block, BS);
}

bool is_pinned(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

int ensure_pinned(Ctx &c, size_t bytes) {
  if (c.pinned_bytes >= bytes) return FW_OK;
  if (c.pinned) cudaFreeHost(c.pinned);
  c.pinned = nullptr;
  c.pinned_bytes = 0;
  if (cudaHostAlloc(&c.pinned, bytes, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    return fail(FW_ENOMEM, "cudaHostAlloc(%zu) failed", bytes);
  }
  c.pinned_bytes = bytes;
  return FW_OK;
}

// Host <-> device copies: direct when the host buffer is pinned, otherwise through two
// pinned staging chunks (copy engine overlaps the host memcpy of the next chunk).
int copy_h2d(Ctx &c, void *dst, const void *src, size_t bytes, cudaStream_t st) {
  if (is_pinned(src)) {
    CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    return FW_OK;
  }
  TRY(ensure_pinned(c, 2 * kStageBytes));
  TRY(ensure_events(c, 4));
  cudaEvent_t done[2] = {c.events[2], c.events[3]};
  bool used[2] = {false, false};
  size_t off = 0;
  for (int b = 0; off < bytes; b ^= 1) {
    const size_t len = std::min(kStageBytes, bytes - off);
    char *stage = static_cast<char *>(c.pinned) + b * kStageBytes;
    if (used[b]) CU(cudaEventSynchronize(done[b]));
    memcpy(stage, static_cast<const char *>(src) + off, len);
    CU(cudaMemcpyAsync(static_cast<char *>(dst) + off, stage, len, cudaMemcpyHostToDevice, st));
    CU(cudaEventRecord(done[b], st));
    used[b] = true;
    off += len;
  }
  return FW_OK;
}

int copy_d2h(Ctx &c, void *dst, const void *src, size_t bytes, cudaStream_t st) {
  if (is_pinned(dst)) {
    CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return FW_OK;
  }
  TRY(ensure_pinned(c, 2 * kStageBytes));
  size_t off = 0;
  for (; off < bytes;) {
    const size_t len = std::min(kStageBytes, bytes - off);
    CU(cudaMemcpyAsync(c.pinned, static_cast<const char *>(src) + off, len, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    memcpy(static_cast<char *>(dst) + off, c.pinned, len);
    off += len;
  }
  return FW_OK;
}

template <typename T>
int solve_host(T *dist, int32_t *next, int64_t n, int block, int ngpus) {
  int BS = 0;
  TRY(check_common(n, dist, block, &BS));
  if (ngpus < 0 || ngpus > 1)
    return fail(FW_EINVAL, "the single-process entry point solves on one GPU (ngpus = 0 or 1); "
                           "multi-GPU runs one process per GPU (paper_1811_01201_b200.dist)");
  Ctx &c = *g_ctx;
  CU(cudaSetDevice(c.dev));
  const size_t bytes = (size_t)n * n * sizeof(T);
  TRY(c.user_d.ensure(bytes));
  if (next) TRY(c.user_t.ensure((size_t)n * n * sizeof(int32_t)));
  T *d = static_cast<T *>(c.user_d.p);
  int32_t *t = next ? static_cast<int32_t *>(c.user_t.p) : nullptr;
  cudaEvent_t h0, h1;
  CU(cudaEventCreate(&h0));
  CU(cudaEventCreate(&h1));
  CU(cudaEventRecord(h0, c.stream));
  int rc = copy_h2d(c, d, dist, bytes, c.stream);
  if (rc == FW_OK) rc = (cudaEventRecord(h1, c.stream) == cudaSuccess) ? FW_OK : FW_ECUDA;
  if (rc == FW_OK) rc = solve_device<T>(c, d, n, t, n, n, BS, c.stream);
  float h2d = 0;
  if (rc == FW_OK) cudaEventElapsedTime(&h2d, h0, h1);
  if (rc == FW_OK) {
    CU(cudaEventRecord(h0, c.stream));
    rc = copy_d2h(c, dist, d, bytes, c.stream);
    if (rc == FW_OK && next) rc = copy_d2h(c, next, t, (size_t)n * n * sizeof(int32_t), c.stream);
    if (rc == FW_OK) {
      CU(cudaEventRecord(h1, c.stream));
      CU(cudaEventSynchronize(h1));
      float d2h = 0;
      cudaEventElapsedTime(&d2h, h0, h1);
      c.stats.h2d_ms = h2d;
      c.stats.d2h_ms = d2h;
    }
  }
  cudaEventDestroy(h0);
  cudaEventDestroy(h1);
  return rc;
}

template <typename T>
int solve_dev_entry(T *d_dist, int32_t *d_next, int64_t n, int64_t ld, int block, void *stream) {
  int BS = 0;
  TRY(check_common(n, d_dist, block, &BS));
  if (ld < n) return fail(FW_EINVAL, "ld (%lld) < n (%lld)", (long long)ld, (long long)n);
  Ctx &c = *g_ctx;
  return solve_device<T>(c, d_dist, ld, d_next, ld, n, BS, static_cast<cudaStream_t>(stream));
}

}  // namespace

extern "C" {

int fw_init(int ngpus_max, unsigned flags) {
  if (g_ctx) return fail(FW_ESTATE, "fw_init called twice without fw_free");
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(FW_ECUDA, "no CUDA device visible");
  }
  if (ngpus_max < 0 || ngpus_max > count)
    return fail(FW_EINVAL, "ngpus_max = %d but %d device(s) visible", ngpus_max, count);
  Ctx *c = new Ctx();
  c->flags = flags;
  CU(cudaGetDevice(&c->dev));
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, c->dev));
  if (prop.major < 10) {
    delete c;
    return fail(FW_ECUDA, "device %s is sm_%d%d; this library is built for sm_100a", prop.name,
                prop.major, prop.minor);
  }
  CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  g_ctx = c;
  g_err.clear();
  return FW_OK;
}

int fw_free(void) {
  if (!g_ctx) return FW_OK;
  Ctx *c = g_ctx;
  cudaDeviceSynchronize();
  c->ws_d.release();
  c->ws_t.release();
  c->user_d.release();
  c->user_t.release();
  c->scratch.release();
  if (c->pinned) cudaFreeHost(c->pinned);
  for (auto e : c->events) cudaEventDestroy(e);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  g_ctx = nullptr;
  return FW_OK;
}

int fw_solve(float *dist, int32_t *next, int64_t n, int block, int ngpus) {
  return solve_host<float>(dist, next, n, block, ngpus);
}

int fw_solve_i32(int32_t *dist, int32_t *next, int64_t n, int block, int ngpus) {
  return solve_host<int32_t>(dist, next, n, block, ngpus);
}

int fw_solve_device_f32(float *d_dist, int32_t *d_next, int64_t n, int64_t ld, int block,
                        void *stream) {
  return solve_dev_entry<float>(d_dist, d_next, n, ld, block, stream);
}

int fw_solve_device_i32(int32_t *d_dist, int32_t *d_next, int64_t n, int64_t ld, int block,
                        void *stream) {
  return solve_dev_entry<int32_t>(d_dist, d_next, n, ld, block, stream);
}

const char *fw_last_error(void) { return g_err.c_str(); }

int fw_last_stats(fw_stats *out) {
  if (!g_ctx || !g_ctx->has_stats) return fail(FW_ESTATE, "no solve has completed yet");
  if (!out) return fail(FW_EINVAL, "out is NULL");
  *out = g_ctx->stats;
  return FW_OK;
}

const char *fw_version(void) { return "fwb200 0.1 sm_100a"; }

}  // extern "C"

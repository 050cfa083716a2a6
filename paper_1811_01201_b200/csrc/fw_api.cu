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
#include <stdlib.h>
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
  cudaStream_t side = nullptr;     // high-priority stream for the look-ahead pivot phases
  bool lookahead = true;
  DevBuf ws_d, ws_t;               // padded workspaces (D, tags/P)
  DevBuf ws_b;                     // backup of W for a speculative key run (in place)
  DevBuf user_d, user_t;           // device copies of host buffers (host entry points)
  DevBuf scratch;                  // validation flags
  void *pinned = nullptr;          // staging for pageable host buffers
  size_t pinned_bytes = 0;
  std::vector<cudaEvent_t> events;
  fw_stats stats{};
  bool has_stats = false;
};

Ctx *g_ctx = nullptr;

constexpr size_t kStageBytes = 64ull << 20;  // pinned staging chunk
// Largest initial/stored distance for which key sums stay exact (kernels header, KEY_*):
// FP32: 2*(T*128+127) < 2^24; INT32: 2*(T*128+127) < FW_INF_I32 (INF + key < 2^31 as well).
constexpr int64_t kKeyMaxF32 = 65534;
constexpr int64_t kKeyMaxI32 = 4194302;

int ensure_events(Ctx &c, size_t count) {
  while (c.events.size() < count) {
    cudaEvent_t e;
    CU(cudaEventCreate(&e));
    c.events.push_back(e);
  }
  return FW_OK;
}

// ---- kernel launch wrappers ---------------------------------------------------------
template <typename T, int TM, int TN, int MODE>
int launch_tile(dim3 grid, cudaStream_t st, T *D, int32_t *P, const TileArgs &a, int *maxkey) {
  constexpr int bytes = TileShape<TM, TN>::kBytes;
  auto kern = grid.z > 1 ? minplus_tile_kernel<T, TM, TN, MODE, true>
                         : minplus_tile_kernel<T, TM, TN, MODE, false>;
  static bool configured = false;  // per instantiation (one device per process)
  if (!configured) {
    CU(cudaFuncSetAttribute(minplus_tile_kernel<T, TM, TN, MODE, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    CU(cudaFuncSetAttribute(minplus_tile_kernel<T, TM, TN, MODE, false>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    configured = true;
  }
  kern<<<grid, kThreads, bytes, st>>>(D, P, a, maxkey);
  CU(cudaGetLastError());
  return FW_OK;
}

TileArgs tile_args(int64_t ld, int kb, int BS, int tag) {
  TileArgs a{};
  a.ld = ld;
  a.kb = kb;
  a.Kd = BS;
  a.tag = tag;
  for (int z = 0; z < 2; ++z) {
    a.mr_lo[z] = a.mr_hi[z] = a.mc_lo[z] = a.mc_hi[z] = 0;
    a.row0[z] = a.col0[z] = a.xrow[z] = 0;
  }
  return a;
}

template <typename T, int BS, int MODE>
int launch_phase1_bs(cudaStream_t st, T *D, int32_t *P, int64_t ld, int kb, int K, int *maxkey) {
  const int bytes = 2 * BS * BS * (int)sizeof(T);   // row-major + transposed copy of D_KK
  auto kern = phase1_kernel<T, BS, MODE>;
  static bool configured = false;
  if (!configured) {
    CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    configured = true;
  }
  kern<<<1, 1024, bytes, st>>>(D, P, ld, kb, K, maxkey);
  CU(cudaGetLastError());
  return FW_OK;
}

template <typename T, int MODE>
int launch_phase1(cudaStream_t st, T *D, int32_t *P, int64_t ld, int kb, int BS, int K, int *maxkey) {
  switch (BS) {
    case 32: return launch_phase1_bs<T, 32, MODE>(st, D, P, ld, kb, K, maxkey);
    case 64: return launch_phase1_bs<T, 64, MODE>(st, D, P, ld, kb, K, maxkey);
    case 128: return launch_phase1_bs<T, 128, MODE>(st, D, P, ld, kb, K, maxkey);
  }
  return fail(FW_EINVAL, "unsupported block size %d", BS);
}

// Phase 2: row strip D[kb:kb+BS, :] and column strip D[:, kb:kb+BS] relaxed
// through the closed diagonal block D_KK* (min-plus product form, reading R7). Both strips
// exclude the diagonal block itself. BS = 128: one launch (blockIdx.z picks the strip).
template <typename T, int MODE, int BS>
int launch_phase2_bs(cudaStream_t st, T *D, int32_t *P, int64_t ld, int64_t n_pad, int kb, int K,
                     int *maxkey) {
  const int tiles = (int)(n_pad / 128);
  TileArgs a = tile_args(ld, kb, BS, K);
  // z = 0: row strip, tiles BS x 128 across the columns; exclude the diagonal block columns
  a.row0[0] = kb; a.col0[0] = 0; a.mc_lo[0] = kb; a.mc_hi[0] = kb + BS;
  // z = 1: column strip, tiles 128 x BS down the rows; exclude the diagonal block rows
  a.row0[1] = 0; a.col0[1] = kb; a.mr_lo[1] = kb; a.mr_hi[1] = kb + BS; a.xrow[1] = 1;
  if (BS == 128) return launch_tile<T, 128, 128, MODE>(dim3(tiles, 1, 2), st, D, P, a, maxkey);
  TileArgs c = a;
  c.row0[0] = 0; c.col0[0] = kb; c.mr_lo[0] = kb; c.mr_hi[0] = kb + BS; c.mc_lo[0] = c.mc_hi[0] = 0;
  c.xrow[0] = 1;
  TRY((launch_tile<T, BS, 128, MODE>(dim3(tiles, 1, 1), st, D, P, a, maxkey)));
  return launch_tile<T, 128, BS, MODE>(dim3(tiles, 1, 1), st, D, P, c, maxkey);
}

template <typename T, int MODE>
int launch_phase2(cudaStream_t st, T *D, int32_t *P, int64_t ld, int64_t n_pad, int kb, int BS,
                  int K, int *maxkey) {
  switch (BS) {
    case 32: return launch_phase2_bs<T, MODE, 32>(st, D, P, ld, n_pad, kb, K, maxkey);
    case 64: return launch_phase2_bs<T, MODE, 64>(st, D, P, ld, n_pad, kb, K, maxkey);
    case 128: return launch_phase2_bs<T, MODE, 128>(st, D, P, ld, n_pad, kb, K, maxkey);
  }
  return fail(FW_EINVAL, "unsupported block size %d", BS);
}

// Phase 3: D_IJ <- min(D_IJ, D_IK (x) D_KJ) for all I != K, J != K.
template <typename T, int MODE>
int launch_phase3(cudaStream_t st, T *D, int32_t *P, int64_t ld, int64_t n_pad, int kb, int BS,
                  int K, int *maxkey) {
  const int tiles = (int)(n_pad / 128);
  TileArgs a = tile_args(ld, kb, BS, K);
  a.mr_lo[0] = a.mc_lo[0] = kb;
  a.mr_hi[0] = a.mc_hi[0] = kb + BS;
  return launch_tile<T, 128, 128, MODE>(dim3(tiles, tiles, 1), st, D, P, a, maxkey);
}

// Look-ahead split of phase 3 (BS = 128). P3a: the tiles of block-row K+1 and block-column
// K+1 (what phases 1-2 of round K+1 read), so round K+1 can start on the side stream while
// P3b — every other tile — finishes round K on the main stream.
template <typename T, int MODE>
int launch_phase3a(cudaStream_t st, T *D, int32_t *P, int64_t ld, int64_t n_pad, int kb, int K,
                   int *maxkey) {
  const int tiles = (int)(n_pad / 128), BS = 128, kn = kb + BS;
  TileArgs a = tile_args(ld, kb, BS, K);
  // z = 0: block-row K+1 across all columns except the column strip of round K
  a.row0[0] = kn; a.col0[0] = 0; a.mc_lo[0] = kb; a.mc_hi[0] = kb + BS;
  // z = 1: block-column K+1 down all rows except the row strip of K and block-row K+1
  a.row0[1] = 0; a.col0[1] = kn; a.mr_lo[1] = kb; a.mr_hi[1] = kn + BS; a.xrow[1] = 1;
  return launch_tile<T, 128, 128, MODE>(dim3(tiles, 1, 2), st, D, P, a, maxkey);
}

template <typename T, int MODE>
int launch_phase3b(cudaStream_t st, T *D, int32_t *P, int64_t ld, int64_t n_pad, int kb, int K,
                   int *maxkey) {
  const int tiles = (int)(n_pad / 128), BS = 128;
  TileArgs a = tile_args(ld, kb, BS, K);
  a.mr_lo[0] = a.mc_lo[0] = kb;            // strips of round K and block-row/column K+1
  a.mr_hi[0] = a.mc_hi[0] = kb + 2 * BS;
  return launch_tile<T, 128, 128, MODE>(dim3(tiles, tiles, 1), st, D, P, a, maxkey);
}

template <typename T>
constexpr bool is_int_v() { return std::is_integral<T>::value; }

struct RoundTimes {
  bool on;
  cudaEvent_t *ev;  // 3 per round: after phase 1, after phase 2, after phase 3
};

// Streams for the look-ahead: phases 1-2 of round K+1 run on `side` while the bulk of
// phase 3 of round K runs on the caller's stream (readings R12).
struct Streams {
  cudaStream_t main, side;
  cudaEvent_t *sync;   // 2 per round
};

template <typename T, int MODE>
int run_rounds(Streams s, T *D, int32_t *P, int64_t ld, int64_t n_pad, int BS, int R, int *maxkey,
               RoundTimes rt, bool lookahead) {
  cudaStream_t st = s.main;
  if (!lookahead || BS != 128 || R < 2) {
    for (int K = 0; K < R; ++K) {
      const int kb = K * BS;
      TRY((launch_phase1<T, MODE>(st, D, P, ld, kb, BS, K, maxkey)));
      if (rt.on) CU(cudaEventRecord(rt.ev[3 * K], st));
      TRY((launch_phase2<T, MODE>(st, D, P, ld, n_pad, kb, BS, K, maxkey)));
      if (rt.on) CU(cudaEventRecord(rt.ev[3 * K + 1], st));
      TRY((launch_phase3<T, MODE>(st, D, P, ld, n_pad, kb, BS, K, maxkey)));
      if (rt.on) CU(cudaEventRecord(rt.ev[3 * K + 2], st));
    }
    return FW_OK;
  }
  // round 0 pivot phases on the main stream
  TRY((launch_phase1<T, MODE>(st, D, P, ld, 0, BS, 0, maxkey)));
  if (rt.on) CU(cudaEventRecord(rt.ev[0], st));
  TRY((launch_phase2<T, MODE>(st, D, P, ld, n_pad, 0, BS, 0, maxkey)));
  if (rt.on) CU(cudaEventRecord(rt.ev[1], st));
  for (int K = 0; K < R; ++K) {
    const int kb = K * BS;
    if (K + 1 < R) {
      TRY((launch_phase3a<T, MODE>(st, D, P, ld, n_pad, kb, K, maxkey)));
      CU(cudaEventRecord(s.sync[2 * K], st));
      // side: phases 1-2 of round K+1 (they only touch block-row/column K+1)
      CU(cudaStreamWaitEvent(s.side, s.sync[2 * K], 0));
      TRY((launch_phase1<T, MODE>(s.side, D, P, ld, kb + BS, BS, K + 1, maxkey)));
      if (rt.on) CU(cudaEventRecord(rt.ev[3 * (K + 1)], s.side));
      TRY((launch_phase2<T, MODE>(s.side, D, P, ld, n_pad, kb + BS, BS, K + 1, maxkey)));
      if (rt.on) CU(cudaEventRecord(rt.ev[3 * (K + 1) + 1], s.side));
      CU(cudaEventRecord(s.sync[2 * K + 1], s.side));
      TRY((launch_phase3b<T, MODE>(st, D, P, ld, n_pad, kb, K, maxkey)));
      if (rt.on) CU(cudaEventRecord(rt.ev[3 * K + 2], st));
      CU(cudaStreamWaitEvent(st, s.sync[2 * K + 1], 0));
    } else {
      TRY((launch_phase3<T, MODE>(st, D, P, ld, n_pad, kb, BS, K, maxkey)));
      if (rt.on) CU(cudaEventRecord(rt.ev[3 * K + 2], st));
    }
  }
  return FW_OK;
}

template <typename T, int MODE>
int run_init(cudaStream_t st, const T *src, int64_t ld_src, int64_t n, T *D, int32_t *P, int64_t ld,
             int64_t n_pad) {
  dim3 g((unsigned)std::min<int64_t>((n_pad + 255) / 256, 64), (unsigned)n_pad);
  init_kernel<T, MODE><<<g, 256, 0, st>>>(src, ld_src, n, D, P, ld, n_pad);
  CU(cudaGetLastError());
  return FW_OK;
}

template <typename T>
int dispatch_init(int mode, cudaStream_t st, const T *src, int64_t ld_src, int64_t n, T *D,
                  int32_t *P, int64_t ld, int64_t n_pad) {
  switch (mode) {
    case MODE_PLAIN: return run_init<T, MODE_PLAIN>(st, src, ld_src, n, D, P, ld, n_pad);
    case MODE_TAG: return run_init<T, MODE_TAG>(st, src, ld_src, n, D, P, ld, n_pad);
    default: return run_init<T, MODE_KEY>(st, src, ld_src, n, D, P, ld, n_pad);
  }
}

template <typename T>
int dispatch_rounds(int mode, Streams s, T *D, int32_t *P, int64_t ld, int64_t n_pad, int BS, int R,
                    int *maxkey, RoundTimes rt, bool lookahead) {
  switch (mode) {
    case MODE_PLAIN: return run_rounds<T, MODE_PLAIN>(s, D, P, ld, n_pad, BS, R, maxkey, rt, lookahead);
    case MODE_TAG: return run_rounds<T, MODE_TAG>(s, D, P, ld, n_pad, BS, R, maxkey, rt, lookahead);
    default: return run_rounds<T, MODE_KEY>(s, D, P, ld, n_pad, BS, R, maxkey, rt, lookahead);
  }
}

// ---- the solve on device buffers ----------------------------------------------------
// src: n rows of ld_src elements (in/out); next: n rows of ld_next int32 or nullptr.
template <typename T>
int solve_device(Ctx &c, T *src, int64_t ld_src, int32_t *next, int64_t ld_next, int64_t n,
                 int BS, cudaStream_t st) {
  const bool int_t = is_int_v<T>();
  const int64_t n_pad = (n + 127) / 128 * 128;
  const bool want_p = next != nullptr;
  const bool lastk = (c.flags & FW_PATH_LAST_K) != 0;
  const int path_mode = want_p ? (lastk ? 1 : 0) : -1;
  const bool timing = (c.flags & FW_TIMING) != 0;

  // 1. validation (read-only; outputs untouched on error)
  TRY(c.scratch.ensure(64));
  int *d_flags = static_cast<int *>(c.scratch.p);   // [0] flags [1] max weight [2] max key
  CU(cudaMemsetAsync(d_flags, 0, 16, st));
  {
    const int64_t total = n * n;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    validate_kernel<T><<<std::max(blocks, 1), 256, 0, st>>>(src, ld_src, n, d_flags, d_flags + 1);
    CU(cudaGetLastError());
  }
  int h_flags[4] = {0, 0, 0, 0};
  CU(cudaMemcpyAsync(h_flags, d_flags, sizeof h_flags, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (h_flags[0] & 1)
    return fail(FW_EINVAL, int_t ? "weight outside [0, FW_INF_I32]" : "negative or NaN weight");
  double maxw;
  if (int_t) {
    maxw = (double)h_flags[1];
  } else {
    float f;
    memcpy(&f, &h_flags[1], 4);
    maxw = f;
  }
  if (int_t && n > 1 && (int64_t)(n - 1) * (int64_t)h_flags[1] >= (int64_t)FW_INF_I32)
    return fail(FW_ERANGE, "(n-1)*max_weight = %lld >= FW_INF_I32: finite path sums could reach INF",
                (long long)(n - 1) * h_flags[1]);

  // 2. P mode: exact arg-min keys for integer-valued data within the key range, else tags
  const int64_t key_max = int_t ? kKeyMaxI32 : kKeyMaxF32;
  const bool integral = int_t || !(h_flags[0] & 2);
  const bool has_inf = (h_flags[0] & 4) != 0;
  int mode = MODE_PLAIN;
  bool key_static = false;
  if (want_p) {
    mode = MODE_TAG;
    if (integral && maxw <= (double)key_max) {
      mode = MODE_KEY;
      // stored finite values never exceed max(W) without INF entries; otherwise a path
      // value is at most (n-1)*max(W) — or is checked after the solve (max stored key)
      key_static = !has_inf || (double)(n - 1) * maxw <= (double)key_max;
    }
  }
  const int key_limit = int_t ? (int)(key_max * 128 + 127) : [] {
    float f = (float)(kKeyMaxF32 * 128 + 127);
    int b;
    memcpy(&b, &f, 4);
    return b;
  }();

  // 3. placement: in place when the caller's buffer already has the padded layout
  const bool inplace = n == n_pad && ld_src == n && ((uintptr_t)src % 16 == 0) &&
                       (!want_p || (ld_next == n && (uintptr_t)next % 16 == 0));
  T *D = src;
  int32_t *Pm = next;
  int64_t ld = n;
  if (!inplace) {
    TRY(c.ws_d.ensure((size_t)n_pad * n_pad * sizeof(T)));
    D = static_cast<T *>(c.ws_d.p);
    if (want_p) {
      TRY(c.ws_t.ensure((size_t)n_pad * n_pad * sizeof(int32_t)));
      Pm = static_cast<int32_t *>(c.ws_t.p);
    }
    ld = n_pad;
  }
  // the speculative key run may have to be redone in TAG mode: keep W when in place
  T *backup = nullptr;
  if (is_key(mode) && !key_static && inplace) {
    TRY(c.ws_b.ensure((size_t)n * n * sizeof(T)));
    backup = static_cast<T *>(c.ws_b.p);
    CU(cudaMemcpyAsync(backup, src, (size_t)n * n * sizeof(T), cudaMemcpyDeviceToDevice, st));
  }

  const int R = (int)((n + BS - 1) / BS);  // rounds wholly inside the padding are skipped
  TRY(ensure_events(c, 4 + 3 * (size_t)R + 2 + 2 * (size_t)R));
  Streams streams{st, c.side, c.events.data() + 4 + 3 * (size_t)R + 2};
  cudaEvent_t e_begin = c.events[0], e_end = c.events[1], e_init = c.events[2],
              e_post = c.events[3];
  RoundTimes rt{timing, c.events.data() + 4};
  int *d_maxkey = d_flags + 2;

  CU(cudaEventRecord(e_begin, st));
  CU(cudaStreamWaitEvent(c.side, e_begin, 0));   // the side stream follows the caller's stream
  for (int attempt = 0; attempt < 2; ++attempt) {
    // 4. init (+ key encoding), rounds
    const T *init_src = (attempt == 1 && backup) ? backup : src;
    const int64_t init_ld = (attempt == 1 && backup) ? n : ld_src;
    TRY(dispatch_init<T>(mode, st, init_src, init_ld, n, D, want_p ? Pm : nullptr, ld, n_pad));
    CU(cudaEventRecord(e_init, st));
    TRY(dispatch_rounds<T>(mode, streams, D, want_p ? Pm : nullptr, ld, n_pad, BS, R, d_maxkey, rt,
                           c.lookahead));
    if (!is_key(mode) || key_static) break;
    CU(cudaMemcpyAsync(h_flags, d_flags, sizeof h_flags, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (h_flags[2] <= key_limit) break;
    mode = MODE_TAG;   // a stored key left the exact range: redo with round tags
    CU(cudaMemsetAsync(d_flags + 2, 0, 4, st));
  }

  // 5. epilogue passes: keys -> distances; tags -> last k; last k -> next hop (R9/R10)
  if (is_key(mode)) {
    dim3 g((unsigned)std::min<int64_t>((n + 255) / 256, 64), (unsigned)n);
    decode_kernel<T><<<g, 256, 0, st>>>(D, ld, n);
    CU(cudaGetLastError());
  }
  if (mode == MODE_TAG) {
    dim3 g((unsigned)((n + 255) / 256), (unsigned)n);
    resolve_lastk_kernel<T><<<g, 256, 0, st>>>(D, ld, Pm, n, BS);
    CU(cudaGetLastError());
  }
  if (want_p) {
    const size_t row_bytes = (size_t)n * sizeof(int32_t);
    const int use_smem = row_bytes <= 200 * 1024;
    static bool configured = false;
    if (!configured) {
      CU(cudaFuncSetAttribute(finalize_paths_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              200 * 1024));
      configured = true;
    }
    finalize_paths_kernel<T><<<(unsigned)n, 1024, use_smem ? row_bytes : 0, st>>>(
        D, Pm, ld, n, path_mode == 0, use_smem, d_flags);
    CU(cudaGetLastError());
  }
  CU(cudaEventRecord(e_post, st));

  // 6. unpad into the caller's buffers
  if (!inplace) {
    dim3 g((unsigned)std::min<int64_t>((n + 255) / 256, 64), (unsigned)n);
    unpad_kernel<T><<<g, 256, 0, st>>>(D, ld, n, src, ld_src);
    CU(cudaGetLastError());
    if (want_p) {
      unpad_kernel<int32_t><<<g, 256, 0, st>>>(Pm, ld, n, next, ld_next);
      CU(cudaGetLastError());
    }
  }
  CU(cudaEventRecord(e_end, st));
  CU(cudaMemcpyAsync(h_flags, d_flags, sizeof h_flags, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (h_flags[0] & 8)
    return fail(FW_ERANGE, "next-hop resolution did not converge (zero-weight cycle?)");

  fw_stats s{};
  s.n = n;
  s.n_pad = n_pad;
  s.block = BS;
  s.rounds = R;
  s.is_int = int_t;
  s.path_mode = path_mode;
  s.p_method = mode;
  float ms = 0.f;
  CU(cudaEventElapsedTime(&ms, e_begin, e_end));
  s.solve_ms = ms;
  s.phase3_launches = R;
  // phase-3 relaxations actually issued: rows and columns outside the round's strips
  double relax = 0;
  for (int K = 0; K < R; ++K) {
    const double off = (double)(n_pad - BS);
    relax += off * off * BS;
  }
  s.phase3_relaxations = relax;
  if (timing) {
    // absolute event times (ms since e_begin); with the look-ahead, phases 1-2 of round K
    // run on the side stream from the end of P3a(K-1), concurrently with P3b(K-1)
    auto at = [&](cudaEvent_t e) {
      float t = 0.f;
      cudaEventElapsedTime(&t, e_begin, e);
      return (double)t;
    };
    const bool la = c.lookahead && BS == 128 && R >= 2;
    const cudaEvent_t *sy = streams.sync;
    double prev_p3_end = at(e_init);
    for (int K = 0; K < R; ++K) {
      const double p1 = at(rt.ev[3 * K]), p2 = at(rt.ev[3 * K + 1]), p3 = at(rt.ev[3 * K + 2]);
      const double p1_start = (la && K > 0) ? at(sy[2 * (K - 1)]) : prev_p3_end;
      s.phase1_ms += p1 - p1_start;
      s.phase2_ms += p2 - p1;
      s.phase3_ms += p3 - std::max(prev_p3_end, p2);
      prev_p3_end = p3;
    }
    s.post_ms = at(e_post) - prev_p3_end;
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
  int prio_lo = 0, prio_hi = 0;
  CU(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  CU(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, prio_hi));
  const char *la = getenv("FW_LOOKAHEAD");
  c->lookahead = !(la && la[0] == '0');
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
  c->ws_b.release();
  c->user_d.release();
  c->user_t.release();
  c->scratch.release();
  if (c->pinned) cudaFreeHost(c->pinned);
  for (auto e : c->events) cudaEventDestroy(e);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->side) cudaStreamDestroy(c->side);
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

// fw_api.cu — C ABI (include/fw.h) and the round driver of the blocked Floyd–Warshall solve
// (arxiv 1811.01201 §4.1), on one GPU or on a block-row partition over
// several GPUs (one process per GPU, NCCL over NVLink).
//
// Round K (the OpenMP structure of P:151-155 becomes stream order):
//   owner(K)  phase 1 on D_KK, phase 2 on its row strip
//   owner(K)  -> all: broadcast of the pivot row strip (BS x n_pad) — the only exchange
//   every GPU phase 2 column strip of its rows (D_KK* comes with the strip)
//   every GPU phase 3 on its rows with A = own column strip, B = the pivot row strip
// Look-ahead (a8): phase 3 of round K is split so that the tiles round K+1's pivot phases
// read are done first (P3a); the pivot phases and broadcast of round K+1 then run on a
// high-priority side stream while the rest of phase 3 (P3b) runs on the main stream.
// After the rounds the post-pass turns keys / round tags into P (reading R9).
// One GPU is the world = 1 case of the same driver (no broadcast: B is read in place); there,
// keyed and distance-only solves take two rounds per phase-3 pass (Rounds::run_pairs,
// DESIGN.md §4.9). The host entry points split the rows into chunks whose copies overlap the
// rounds (solve_host_pipelined, reading R16).
#include "fw_kernels.cuh"
#include "fw_persist.cuh"
#include "../../include/fw.h"

#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <map>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <type_traits>
#include <utility>
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

// ---- NCCL, loaded on first use (the libnccl.so.2 torch has already loaded, when present) ----
struct Nccl {
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t *, int, const int *) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommInitRankConfig)(ncclComm_t *, int, ncclUniqueId, int, ncclConfig_t *) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
};
Nccl g_nccl;

int load_nccl() {
  if (g_nccl.h) return FW_OK;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return fail(FW_ENCCL, "cannot load libnccl.so.2: %s", dlerror());
#define SYM(name)                                                                        \
  *reinterpret_cast<void **>(&g_nccl.name) = dlsym(h, "nccl" #name);                     \
  if (!g_nccl.name) return fail(FW_ENCCL, "libnccl.so.2 lacks nccl" #name);
  SYM(GetUniqueId) SYM(CommInitRank) SYM(CommInitAll) SYM(CommDestroy) SYM(Broadcast) SYM(AllReduce) SYM(AllGather)
  SYM(GroupStart) SYM(GroupEnd) SYM(GetErrorString) SYM(CommInitRankConfig) SYM(CommGetAsyncError)
  SYM(CommAbort)
#undef SYM
  g_nccl.h = h;
  return FW_OK;
}

#define NC(call)                                                                          \
  do {                                                                                    \
    ncclResult_t r_ = (call);                                                             \
    if (r_ != ncclSuccess)                                                                \
      return fail(FW_ENCCL, "%s failed: %s", #call, g_nccl.GetErrorString(r_));           \
  } while (0)

// ---- device / host buffers --------------------------------------------------------------
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
  DevBuf ws_d, ws_t;               // padded local workspaces (D, tags/P)
  DevBuf ws_b;                     // backup of W for a speculative key run (in place)
  DevBuf ws_s;                     // two pivot-strip receive buffers (multi-GPU)
  DevBuf ws_tr;                    // transposed final D (round tags only)
  DevBuf user_d, user_t;           // device copies of host buffers (host entry points)
  DevBuf scratch;                  // flags / reductions
  void *pinned = nullptr;          // staging for pageable host buffers
  int *pin_small = nullptr;        // host pipeline: per-chunk max-key snapshots (pinned)
  std::vector<cudaEvent_t> ring_ev; // staging ring (pageable host buffers): last copy per slot
  std::vector<bool> ring_used;
  int ring_pos = 0;
  size_t pinned_bytes = 0;
  std::vector<cudaEvent_t> events;
  cudaStream_t copy = nullptr;     // host pipeline: H2D / D2H of row chunks
  std::vector<cudaEvent_t> pev;    // host pipeline: per-chunk landed / finished events
  int pipe_tiles = -1;             // host pipeline chunk in tile-rows (-1 auto, 0 off)
  int pipe_first = 8;              // auto geometry: first chunk (tile-rows; env FW_PIPE_FIRST)
  bool pairs = true;               // two rounds per phase-3 pass for keyed / plain solves (env FW_PAIRS=0: off)
  bool pair_pdl = true;            // pairs: bulk launches programmatically serialized (env FW_PDL=0: off)
  bool last_pdl = false;           // the last solve's pairs ran with programmatic serialization
  std::vector<cudaEvent_t> xev;    // disable-timing events between bulk launches
  std::vector<cudaStream_t> lb_st; // loopback transport: main and look-ahead stream of every emulated rank
  std::vector<cudaEvent_t> lb_ev;  // loopback transport: disable-timing fork / join / broadcast events
  bool pair_order = true;          // pairs: the next pair's strips run beside the bulk launch (env FW_PAIR_ORDER=0: before it)
  int pipe_pair_rows = 32;         // host pipeline: smallest chunk (tile-rows) run in pairs (env FW_PIPE_PAIR_ROWS)
  bool last_pairs = false;         // the last solve ran in pairs (stats layout)
  int persistent = -1;             // one persistent launch per solve (fw_persist.cuh): -1 auto, 0 off, 1 on
  int persist_gap = -1;            // persistent: rest tiles between P1(K+1) and P2(K+1) (-1 auto)
  int persist_relaxed = 0;         // persistent: dependency polls with relaxed loads (A/B option)
  int persist_stage_old = 1;       // persistent: 128 x 128 tiles stage their old values in shared memory
  int persist_p1_lone = -1;        // persistent, one GPU: every P1 item on one CTA alone on its SM
                                   // (-1 auto = on: C2 5.74 -> 5.52 ms; 0 off, 1 on)
  int persist_quarters = -1;       // persistent, one GPU: critical-path tiles as 64 x 64 quarter items
                                   // (-1 auto: when T < 32 tiles per side, i.e. n < 4096)
  bool last_persist = false;       // the last solve ran as one persistent launch
  bool async = false;              // device entry: no validation, no host synchronisation (fw_set_option)
  bool in_host_entry = false;      // inside fw_solve / fw_solve_i32 (async never applies there)
  bool pending = false;            // an async solve's stats are completed by fw_last_stats
  cudaStream_t pending_st = nullptr;
  DevBuf ws_ver;                   // persistent: per-tile round counters, pub flags, work counter, items
  DevBuf ws_ring;                  // persistent: pivot-row ring(s) (n_pad^2 each) [+ pub flags, NCCL mode]
  DevBuf ws_ipc;                   // persistent NCCL mode: all-gathered IPC handles
  struct Nvls {                    // persistent NCCL mode: the rings as ONE multicast object (NVLS)
    bool active = false;
    CUmemGenericAllocationHandle mc = 0, mem = 0;
    CUdeviceptr uc = 0, mcva = 0;  // this rank's ring (unicast) and the multicast address of all rings
    size_t size = 0;
    int world = 0;
  } nvls;
  int nvls_opt = -1;               // -1: the multicast publish when W > 1 and every device supports it,
                                   // 0: never, 1: also try with one rank (tests the setup / fallback)
  bool last_nvls = false;          // the last solve published through the multicast object
  std::vector<void *> peer_ring;   // persistent NCCL mode: the peers' rings, IPC-mapped
  std::vector<cudaIpcMemHandle_t> peer_handle;
  ncclComm_t comm = nullptr;       // multi-GPU communicator (fw_comm_init, or the team's)
  bool comm_dead = false;          // the communicator was aborted (error, timeout, failed peer)
  std::atomic<int> *abort_flag = nullptr;   // team solve: set by the first rank that fails
  int rank = 0, world = 1;
  int ngpus_max = 1;               // fw_init's limit (0 there = every visible device)
  std::vector<Ctx *> team;         // fw_solve with ngpus > 1: one context per device, rank = device
  fw_stats stats{};
  bool has_stats = false;
};

Ctx *g_ctx = nullptr;
// kernels this library launched (fw_stats.kernel_launches); per host thread, so the rank
// threads of a single-process multi-GPU solve count their own launches
thread_local int64_t g_launches = 0;

// NCCL broadcasts this thread issued (fw_stats.broadcasts / bcast_bytes)
thread_local int64_t g_bcasts = 0;
thread_local double g_bcast_bytes = 0;

// ---- NCCL failure handling --------------------------------------------------------------
// Communicators are created non-blocking (ncclConfig_t.blocking = 0): no NCCL call blocks the
// host, a call may return ncclInProgress and is then polled to completion here. Every wait of
// a multi-GPU solve (NCCL calls, stream synchronisation) is bounded: it polls
// ncclCommGetAsyncError, the team's abort flag (a rank of a single-process team failed) and a
// timeout (env FW_NCCL_TIMEOUT_MS, default 600000), and on any of them aborts the communicator
// (its kernels exit) so the call returns FW_ENCCL instead of hanging.
int64_t nccl_timeout_ms() {
  const char *e = getenv("FW_NCCL_TIMEOUT_MS");
  const long long v = e ? atoll(e) : 0;
  return v > 0 ? v : 600000;
}

int comm_abort(Ctx &c, const char *why) {
  if (c.comm) g_nccl.CommAbort(c.comm);
  c.comm = nullptr;
  c.comm_dead = true;
  if (c.abort_flag) c.abort_flag->store(1);
  return fail(FW_ENCCL, "NCCL communicator aborted: %s", why);
}

bool peer_failed(const Ctx &c) { return c.abort_flag && c.abort_flag->load() != 0; }

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// One poll of the communicator's state: FW_OK while healthy (done or still in progress).
int comm_health(Ctx &c, bool *in_progress, std::chrono::steady_clock::time_point t0, const char *what) {
  ncclResult_t st = ncclSuccess;
  const ncclResult_t r = g_nccl.CommGetAsyncError(c.comm, &st);
  if (r != ncclSuccess) st = r;
  *in_progress = st == ncclInProgress;
  char buf[320];
  if (st != ncclSuccess && st != ncclInProgress) {
    snprintf(buf, sizeof buf, "%s: %s", what, g_nccl.GetErrorString(st));
    return comm_abort(c, buf);
  }
  if (peer_failed(c)) {
    snprintf(buf, sizeof buf, "%s: another rank of the team failed", what);
    return comm_abort(c, buf);
  }
  if (ms_since(t0) > (double)nccl_timeout_ms()) {
    snprintf(buf, sizeof buf, "%s: timed out after %lld ms (FW_NCCL_TIMEOUT_MS)", what,
             (long long)nccl_timeout_ms());
    return comm_abort(c, buf);
  }
  return FW_OK;
}

// Poll a non-blocking communicator until its pending operation (init, enqueue) has completed.
int nccl_settle(Ctx &c, const char *what) {
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    bool busy = false;
    TRY(comm_health(c, &busy, t0, what));
    if (!busy) return FW_OK;
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

// NCCL call on the context's communicator (ncclInProgress polled, errors abort it).
#define NCC(c, call)                                                                              \
  do {                                                                                            \
    if (!(c).comm) return fail(FW_ENCCL, "no live NCCL communicator for %s", #call);             \
    const ncclResult_t r_ = (call);                                                               \
    if (r_ == ncclInProgress) TRY(nccl_settle((c), #call));                                       \
    else if (r_ != ncclSuccess) {                                                                 \
      char b_[320];                                                                               \
      snprintf(b_, sizeof b_, "%s: %s", #call, g_nccl.GetErrorString(r_));                        \
      return comm_abort((c), b_);                                                                 \
    }                                                                                             \
  } while (0)

// Wait for a stream. With a communicator (or inside a team solve) the wait polls: a hung or
// failed collective, or a failed peer, aborts the communicator and returns FW_ENCCL.
int sync_stream(Ctx &c, cudaStream_t st) {
  if (!c.comm && !c.abort_flag) {
    CU(cudaStreamSynchronize(st));
    return FW_OK;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t e = cudaStreamQuery(st);
    if (e == cudaSuccess) return FW_OK;
    if (e != cudaErrorNotReady) CU(e);
    if (c.comm) {
      bool busy = false;
      TRY(comm_health(c, &busy, t0, "waiting for the solve's stream"));
    } else if (peer_failed(c)) {
      return fail(FW_ENCCL, "another rank of the team failed");
    } else if (ms_since(t0) > (double)nccl_timeout_ms()) {
      return fail(FW_ENCCL, "stream wait timed out (FW_NCCL_TIMEOUT_MS)");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

// NVTX ranges (host-side enqueue spans per solve / round or pair / pivot phases / broadcast,
// for an nsys timeline: the GPU work of a range is what it enqueued).
struct Nvtx {
  explicit Nvtx(const char *name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

// Dynamic shared memory limits are a per-device function attribute: set once per
// (kernel, device) — a process may drive several devices (fw_solve with ngpus > 1).
std::mutex g_attr_mu;
std::map<std::pair<const void *, int>, int> g_attr_done;

int smem_attr(const void *fn, int bytes) {
  int dev = 0;
  CU(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_attr_mu);
  int &have = g_attr_done[{fn, dev}];
  if (have >= bytes) return FW_OK;
  CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  have = bytes;
  return FW_OK;
}

// Largest initial/stored distance for which key sums stay exact (kernels header, KEY mode):
// FP32: 2*(T*256+255) < 2^24; INT32: 2*(T*256+255) < FW_INF_I32 (INF + key < 2^31 as well).
constexpr int64_t kKeyMaxF32 = 32766;
constexpr int64_t kKeyMaxI32 = 2097150;

int ensure_xev(Ctx &c, size_t count) {
  while (c.xev.size() < count) {
    cudaEvent_t e;
    CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c.xev.push_back(e);
  }
  return FW_OK;
}

int ensure_events(Ctx &c, size_t count) {
  while (c.events.size() < count) {
    cudaEvent_t e;
    CU(cudaEventCreate(&e));
    c.events.push_back(e);
  }
  return FW_OK;
}

// ---- block-row partition (SURVEY §8 e) ------------------------------------------------------
// The n_pad/128 tile rows are split into `world` contiguous ranges whose sizes differ by at
// most one tile row; rank r owns global rows [row0, row0 + nrows) of the padded matrix.
void partition(int64_t n, int world, int rank, int64_t *row0, int64_t *nrows) {
  const int64_t tiles = (n + 127) / 128;
  const int64_t base = tiles / world, rem = tiles % world;
  const int64_t t0 = rank * base + std::min<int64_t>(rank, rem);
  const int64_t cnt = base + (rank < rem ? 1 : 0);
  *row0 = t0 * 128;
  *nrows = cnt * 128;
}

int owner_of(int64_t n, int world, int64_t row) {
  for (int r = 0; r < world; ++r) {
    int64_t r0, nr;
    partition(n, world, r, &r0, &nr);
    if (row >= r0 && row < r0 + nr) return r;
  }
  return -1;
}

// ---- kernel launch wrappers ----------------------------------------------------------------
template <typename T, int TM, int TN, int MODE>
int launch_tile(dim3 grid, cudaStream_t st, T *D, int32_t *P, const TileArgs &a, int *maxkey, bool pdl = false) {
  if (grid.x == 0 || grid.y == 0) return FW_OK;
  constexpr int bytes = TileShape<TM, TN>::kBytes;
  auto kern = grid.z > 1 ? minplus_tile_kernel<T, TM, TN, MODE, true>
                         : minplus_tile_kernel<T, TM, TN, MODE, false>;
  TRY(smem_attr((const void *)kern, bytes));
  if (pdl) {   // programmatic serialization with the previous launch in st (see the kernel)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CU(cudaLaunchKernelEx(&cfg, kern, D, P, a, maxkey));
    ++g_launches;
    return FW_OK;
  }
  kern<<<grid, kThreads, bytes, st>>>(D, P, a, maxkey);
  ++g_launches;
  CU(cudaGetLastError());
  return FW_OK;
}

// One strip description (z slot) of a tile launch: tile grid origin (local row, global
// column), excluded local rows [mr_lo, mr_hi) and global columns [mc_lo, mc_hi), and whether
// blockIdx.x walks tile rows (a column strip sharing a launch with a row strip).
struct Strip {
  int row0, col0, mr_lo, mr_hi, mc_lo, mc_hi, xrow;
};

TileArgs tile_args(int64_t ld, const void *B, int64_t ldb, int kb, int BS, int tag, int64_t rows,
                   int64_t cols) {
  TileArgs a{};
  a.ld = ld;
  a.rows_lim = (int)rows;
  a.cols_lim = (int)cols;
  a.B = B;
  a.ldb = ldb;
  a.kb = kb;
  a.Kd = BS;
  a.tag = tag;
  return a;
}

void put(TileArgs &a, int z, const Strip &s) {
  a.row0[z] = s.row0; a.col0[z] = s.col0; a.mr_lo[z] = s.mr_lo; a.mr_hi[z] = s.mr_hi;
  a.mc_lo[z] = s.mc_lo; a.mc_hi[z] = s.mc_hi; a.xrow[z] = s.xrow;
}

// phase 1 at BS = 128 as the blocked closure (phase1_blocked_body / _key_body): the persistent
// kernel's phase-1 items use it by default (C2 persistent 6.49 -> 6.10 ms: the pair body spills
// inside that kernel), the stream-ordered launches keep the pair-step kernels, which are faster
// alone (isolated, per round: round tags 39.6 vs 41.9 us, FP32 keys 53.9 vs 61.7 us;
// profiles/r02_p1_blocked_ab.jsonl). Env FW_P1_BLOCKED=0/1 forces either everywhere (A/B).
int g_p1_blocked = -1;

template <typename T, int BS, int MODE>
int launch_phase1_bs(cudaStream_t st, T *D, int32_t *P, int64_t ld, int r0, int kb, int K,
                     int *maxkey) {
  // the tile lives in registers; shared memory holds only row / column k (static, 2 KB at BS = 128),
  // so the CTA fits beside a phase-3 CTA on one SM (the look-ahead starts it early)
  // 256 threads of (BS/16)^2 elements (512 threads of 8 x 4 or 4 x 8 at BS = 128 measured slower:
  // C2 TAG 39.6 -> 48.3 / 47.0 us, C4 keys 55.1 -> 59.9 / 58.0 us per round)
  if constexpr (BS == 128 && is_key(MODE) && std::is_same<T, float>::value) {
    if (g_p1_blocked == 1) {   // FP32 keys: the blocked closure on keys
      TRY(smem_attr((const void *)phase1_blocked_key_kernel, (int)sizeof(P1BSmem<float>)));
      phase1_blocked_key_kernel<<<1, 256, sizeof(P1BSmem<float>), st>>>(reinterpret_cast<float *>(D), P, ld, r0,
                                                                         kb, maxkey);
      ++g_launches;
      CU(cudaGetLastError());
      return FW_OK;
    }
  }
  if constexpr (BS == 128 && !is_key(MODE)) {
    if (g_p1_blocked == 1) {   // PLAIN / TAG: the blocked closure (4 sub-rounds of 32)
      auto kern = phase1_blocked_kernel<T, MODE>;
      TRY(smem_attr((const void *)kern, (int)sizeof(P1BSmem<T>)));
      kern<<<1, 256, sizeof(P1BSmem<T>), st>>>(D, P, ld, r0, kb, K);
      ++g_launches;
      CU(cudaGetLastError());
      return FW_OK;
    }
  }
  constexpr int R1 = BS / kP1Side;
  if (std::is_same<T, float>::value && is_key(MODE)) {   // FP32 keys: select-free variant
    phase1_key_f32_kernel<BS, R1, R1><<<1, kP1Side * kP1Side, 0, st>>>(reinterpret_cast<float *>(D), P, ld, r0, kb,
                                                                      maxkey);
  } else if (!is_key(MODE)) {                             // PLAIN / TAG: two steps per barrier
    phase1_pair_kernel<T, BS, is_key(MODE) ? MODE_PLAIN : MODE, R1, R1><<<1, kP1Side * kP1Side, 0, st>>>(D, P, ld,
                                                                                                       r0, kb, K);
  } else {                                                // INT32 keys: per-step P select
    phase1_kernel<T, BS, MODE><<<1, kP1Side * kP1Side, 0, st>>>(D, P, ld, r0, kb, K, maxkey);
  }
  ++g_launches;
  CU(cudaGetLastError());
  return FW_OK;
}

// Per-round event slots: 3 per round (after phase 1, after phase 2, after phase 3) and 2
// look-ahead synchronisation events per round.
struct Events {
  bool timing;
  cudaEvent_t *ev;
  cudaEvent_t *sync;
};

// The rounds of one GPU's rows (local rows [0, nrows) = global [row0, row0 + nrows)).
template <typename T, int MODE>
struct Rounds {
  Ctx &c;
  int world;     // ranks of the partition (1, the NCCL communicator, or loopback parts)
  T *D;
  int32_t *P;
  int64_t ld, n, n_pad, row0, nrows;
  int BS, R;
  int *maxkey;
  T *strip[2];   // receive buffers of the pivot row strip (world > 1)
  int *done;     // R look-ahead tile counters (zeroed per solve)
  const T *Dg = nullptr;   // one GPU, a row range of the matrix (host pipeline): global row 0,
                           // so the pivot strips of other rows are read in place

  // d_flags of the solve: maxkey is always d_flags + 2; bit 4 of d_flags[0] = a look-ahead
  // wait timed out (wait_count_kernel)
  int *errflags() const { return maxkey - 2; }
  int wait_count(cudaStream_t st, int K, int target) {
    wait_count_kernel<<<1, 1, 0, st>>>(done + K, target, errflags(), 20ull * 1000 * 1000 * 1000);
    ++g_launches;
    CU(cudaGetLastError());
    return FW_OK;
  }

  bool owns(int K) const {
    const int64_t kb = (int64_t)K * BS;
    return kb >= row0 && kb < row0 + nrows;
  }
  int lrow(int K) const { return (int)((int64_t)K * BS - row0); }
  // B operand of round K: the pivot row strip (global rows kb..kb+BS), read in place on its
  // owner and from the broadcast buffer elsewhere
  const T *bstrip(int K) const {
    if (owns(K)) return D + (int64_t)lrow(K) * ld;
    if (Dg) return Dg + (int64_t)K * BS * ld;
    return world == 1 ? D + (int64_t)lrow(K) * ld : strip[K & 1];
  }

  int phase1(cudaStream_t st, int K) {
    if (!owns(K)) return FW_OK;
    switch (BS) {
      case 32: return launch_phase1_bs<T, 32, MODE>(st, D, P, ld, lrow(K), K * BS, K, maxkey);
      case 64: return launch_phase1_bs<T, 64, MODE>(st, D, P, ld, lrow(K), K * BS, K, maxkey);
      default: return launch_phase1_bs<T, 128, MODE>(st, D, P, ld, lrow(K), K * BS, K, maxkey);
    }
  }

  // Phase 2: row strip (owner) and column strip (local rows) relaxed through the
  // closed diagonal block D_KK* (product form, reading R7); the diagonal block is excluded.
  template <int B>
  int phase2_bs(cudaStream_t st, int K, bool row_strip, bool col_strip) {
    const int kb = K * B, tiles_c = (int)(n_pad / 128), tiles_r = (int)(nrows / 128);
    TileArgs a = tile_args(ld, bstrip(K), ld, kb, B, K, nrows, n_pad);
    const bool own = owns(K);
    const int lr = own ? lrow(K) : 0;
    const Strip row{lr, 0, 0, 0, kb, kb + B, 0};                          // B x 128 tiles
    const Strip col{0, kb, own ? lr : 0, own ? lr + B : 0, 0, 0, 1};      // 128 x B tiles
    row_strip = row_strip && own;
    if (B == 128 && row_strip && col_strip) {
      put(a, 0, row);
      put(a, 1, col);
      return launch_tile<T, 128, 128, MODE>(dim3(std::max(tiles_c, tiles_r), 1, 2), st, D, P, a,
                                            maxkey);
    }
    // a single strip (multi-GPU: the owner's row strip before the broadcast, every rank's column
    // strip after it — both on the per-round critical path): at BS = 128 half-width tiles, twice
    // the CTAs with half the work each. Row-strip tiles keep all 128 pivot rows (B is the tile's
    // own columns), column-strip tiles all 128 block columns (A is the tile's own rows), so no
    // CTA reads what another writes.
    if (row_strip) {
      put(a, 0, row);
      if (B == 128) TRY((launch_tile<T, 128, 64, MODE>(dim3(2 * tiles_c, 1, 1), st, D, P, a, maxkey)));
      else TRY((launch_tile<T, B, 128, MODE>(dim3(tiles_c, 1, 1), st, D, P, a, maxkey)));
    }
    if (col_strip) {
      put(a, 0, col);
      if (B == 128) TRY((launch_tile<T, 64, 128, MODE>(dim3(2 * tiles_r, 1, 1), st, D, P, a, maxkey)));
      else TRY((launch_tile<T, 128, B, MODE>(dim3(tiles_r, 1, 1), st, D, P, a, maxkey)));
    }
    return FW_OK;
  }
  int phase2(cudaStream_t st, int K, bool row_strip, bool col_strip) {
    switch (BS) {
      case 32: return phase2_bs<32>(st, K, row_strip, col_strip);
      case 64: return phase2_bs<64>(st, K, row_strip, col_strip);
      default: return phase2_bs<128>(st, K, row_strip, col_strip);
    }
  }

  // Phase 3 on the local rows except rows [rx_lo, rx_hi) and columns [cx_lo, cx_hi).
  int phase3(cudaStream_t st, int K, int rx_lo, int rx_hi, int cx_lo, int cx_hi, bool pdl = false) {
    TileArgs a = tile_args(ld, bstrip(K), ld, K * BS, BS, K, nrows, n_pad);
    put(a, 0, Strip{0, 0, rx_lo, rx_hi, cx_lo, cx_hi, 0});
    return launch_tile<T, 128, 128, MODE>(dim3((unsigned)(n_pad / 128), (unsigned)(nrows / 128), 1),
                                          st, D, P, a, maxkey, pdl);
  }
  int phase3_full(cudaStream_t st, int K, bool pdl = false) {
    const int kb = K * BS;
    const bool own = owns(K);
    return phase3(st, K, own ? lrow(K) : 0, own ? lrow(K) + BS : 0, kb, kb + BS, pdl);
  }

  // Rounds [K0, K1) whose pivot strips (rows of other chunks, read in place through Dg) have
  // completed those rounds (host pipeline, BS = 128, reading R16): no pivot phases, so each
  // round is one phase-3 launch that leaves the round's own column block alone, and the
  // column-strip products of all K1 - K0 blocks follow in one launch (colstrip mode). The
  // column-strip update may come after later rounds: phase 3 of round K reaches every path
  // through block K via its FIRST block-K vertex u (D[i][u] needs no block-K intermediate,
  // D[u][j] is complete), and the strip's own elements only need it before these rows' next
  // pivot phases or their end.
  // With pairs (keyed / plain, BS = 128): rounds K, K+1 (K even) share one 256-deep launch that
  // leaves both column blocks alone; those blocks then take, after the own-block strip batch, the
  // partner block too (colstrip = 2: even blocks through their odd partner, then odd through
  // even, so no launch reads a tile it writes). Same argument: with pivots complete for both
  // rounds, the first block-K or block-K+1 vertex of a path is reached from unrelaxed operands.
  int run_plain(cudaStream_t st, int K0, int K1, bool pairs = false) {
    if (K0 >= K1 || nrows == 0) return FW_OK;
    pairs = pairs && BS == 128 && MODE != MODE_TAG;
    int fused0 = -1, fused1 = -1;          // blocks [fused0, fused1) went through in pairs
    for (int K = K0; K < K1; ++K) {
      const int kb = K * BS;
      if (pairs && K % 2 == 0 && K + 1 < K1) {
        TileArgs a = tile_args(ld, bstrip(K), ld, kb, 2 * BS, K, nrows, n_pad);
        put(a, 0, Strip{0, 0, 0, 0, kb, kb + 2 * BS, 0});
        TRY((launch_tile<T, 128, 128, MODE>(dim3((unsigned)(n_pad / 128), (unsigned)(nrows / 128), 1), st, D, P,
                                            a, maxkey)));
        if (fused0 < 0) fused0 = K;
        fused1 = K + 2;
        ++K;
        continue;
      }
      TRY(phase3(st, K, 0, 0, kb, kb + BS));
    }
    TileArgs a = tile_args(ld, Dg, ld, 0, BS, 0, nrows, n_pad);
    a.colstrip = 1;
    put(a, 0, Strip{0, K0 * BS, 0, 0, 0, 0, 0});
    TRY((launch_tile<T, 128, 128, MODE>(dim3((unsigned)(K1 - K0), (unsigned)(nrows / 128), 1), st, D, P, a,
                                        maxkey)));
    if (fused0 < 0) return FW_OK;
    for (int par = 0; par < 2; ++par) {     // even blocks through their partner, then odd ones
      TileArgs x = tile_args(ld, Dg, ld, 0, BS, 0, nrows, n_pad);
      x.colstrip = 2;
      x.colstep = 2;
      put(x, 0, Strip{0, (fused0 + par) * BS, 0, 0, 0, 0, 0});
      TRY((launch_tile<T, 128, 128, MODE>(dim3((unsigned)((fused1 - fused0) / 2), (unsigned)(nrows / 128), 1), st,
                                          D, P, x, maxkey)));
    }
    return FW_OK;
  }

  // Look-ahead (BS = 128): one ordered phase-3 launch per round whose first nprio CTAs are
  // the tiles round K+1's pivot phases read (block-row K+1 if local, block-column K+1 of the
  // local rows); they count themselves into done[K] and the pivot stream waits on that count
  // (wait_count_kernel) instead of a kernel boundary.
  int phase3_ordered(cudaStream_t st, int K, int *done, int *nprio_out, bool pdl = false) {
    TileArgs a = tile_args(ld, bstrip(K), ld, K * BS, BS, K, nrows, n_pad);
    a.order = 1;
    a.tiles_r = (int)(nrows / 128);
    a.tiles_c = (int)(n_pad / 128);
    a.rowK = owns(K) ? lrow(K) / 128 : -1;
    a.rowN = owns(K + 1) ? lrow(K + 1) / 128 : -1;
    a.colK = K;
    a.colN = K + 1;
    const int nA1 = a.rowN >= 0 ? a.tiles_c - 1 : 0;
    const int rows_b = a.tiles_r - (a.rowK >= 0) - (a.rowN >= 0);
    a.nprio = nA1 + rows_b;
    a.done = done;
    *nprio_out = a.nprio;
    const int64_t total = (int64_t)nA1 + rows_b + (int64_t)rows_b * (a.tiles_c - 2);
    return launch_tile<T, 128, 128, MODE>(dim3((unsigned)total, 1, 1), st, D, P, a, maxkey, pdl);
  }

  // ---- two rounds per phase-3 pass (keyed / plain solves, one GPU, all rows, BS = 128) ------
  // Pair Pp = rounds a = 2Pp, b = a + 1. Its strip region (block-rows and
  // block-columns a, b) is brought through both rounds by two sub-rounds of the usual pivot
  // phases plus one restricted phase-3 launch each (strip3); every other tile then relaxes
  // through blocks a and b in ONE 256-deep product (pair_bulk) — the sequential result, since A
  // (columns a, b) and B (rows a, b) have completed both rounds — with one epilogue instead of
  // two. The next pair's strips go first (pair_prio) so its pivot phases run on the side stream
  // under the bulk launch.
  int strip3(cudaStream_t st, int x, int y) {   // row y (columns != x) and column y (rows != x, y) through block x
    const int kb = x * BS, tiles_c = (int)(n_pad / 128), tiles_r = (int)(nrows / 128);
    TileArgs t = tile_args(ld, D + (int64_t)lrow(x) * ld, ld, kb, BS, x, nrows, n_pad);
    const int lo = lrow(std::min(x, y));    // local rows (the pipeline's row ranges)
    put(t, 0, Strip{lrow(y), 0, 0, 0, kb, kb + BS, 0});
    put(t, 1, Strip{0, y * BS, lo, lo + 2 * BS, 0, 0, 1});
    return launch_tile<T, 128, 128, MODE>(dim3(std::max(tiles_c, tiles_r), 1, 2), st, D, P, t, maxkey);
  }
  int pair_pivot(cudaStream_t st, int Pp) {
    const int a = 2 * Pp, b = a + 1;
    TRY(phase1(st, a));
    TRY(phase2(st, a, true, true));
    TRY(strip3(st, a, b));
    TRY(phase1(st, b));
    TRY(phase2(st, b, true, true));
    return strip3(st, b, a);
  }
  // B operand of pair Pp: rows a, b = 2Pp, 2Pp+1 (both rounds complete) — in place on their
  // owner (one GPU: always; host pipeline: through Dg), the broadcast buffer elsewhere
  const T *bpair(int Pp) const {
    const int a = 2 * Pp;
    if (owns(a) || Dg || world == 1) return D + (int64_t)lrow(a) * ld;
    return strip[Pp & 1];
  }
  int pair_prio(cudaStream_t st, int Pp) {   // rows / columns c, d = a+2, a+3 through blocks a, b
    const int a = 2 * Pp, c2 = a + 2, kb = a * BS;
    const int tiles_c = (int)(n_pad / 128), tiles_r = (int)(nrows / 128);
    TileArgs t = tile_args(ld, bpair(Pp), ld, kb, 2 * BS, a, nrows, n_pad);
    // rows c, d (grid.y = 2) when they are this rank's (else a row origin past the local rows:
    // every tile of that strip exits), then columns c, d of the local rows outside a..d (the
    // exclusion is in local row numbers; it misses the local rows when a..d are another rank's)
    put(t, 0, Strip{owns(c2) || Dg || world == 1 ? lrow(c2) : (int)nrows, 0, 0, 0, kb, kb + 2 * BS, 0});
    put(t, 1, Strip{0, c2 * BS, lrow(a), lrow(a) + 4 * BS, 0, 0, 1});
    return launch_tile<T, 128, 128, MODE>(dim3(std::max(tiles_c, tiles_r), 2, 2), st, D, P, t, maxkey);
  }
  // Non-owner ranks of pair Pp (block-row partition): bring the local columns a, b through both
  // rounds with B = the received rows a, b (final for both rounds). Exact (reading R16): a
  // shortest i -> v path (v in a or b) through blocks <= b has a first vertex u in a or b, and
  // D[u][v] is final, so relaxing (i, a) through a and (i, b) through b, then (i, a) through b
  // with the new (i, b), then (i, b) through a with the new (i, a) reaches it — three launches
  // (colstrip 1: each column block through itself; colstrip 2: through its partner, even blocks
  // first, so no launch reads a tile it writes), the host pipeline's column-strip batch.
  int pair_cols(cudaStream_t st, int Pp) {
    const int a = 2 * Pp;
    const T *B0 = strip[Pp & 1] - (int64_t)a * BS * ld;   // row 0 of a virtual matrix: rows a, b at a*BS
    TileArgs x = tile_args(ld, B0, ld, 0, BS, 0, nrows, n_pad);
    x.colstrip = 1;
    put(x, 0, Strip{0, a * BS, 0, 0, 0, 0, 0});
    TRY((launch_tile<T, 128, 128, MODE>(dim3(2, (unsigned)(nrows / 128), 1), st, D, P, x, maxkey)));
    for (int par = 0; par < 2; ++par) {
      TileArgs y = tile_args(ld, B0, ld, 0, BS, 0, nrows, n_pad);
      y.colstrip = 2;
      y.colstep = 2;
      put(y, 0, Strip{0, (a + par) * BS, 0, 0, 0, 0, 0});
      TRY((launch_tile<T, 128, 128, MODE>(dim3(1, (unsigned)(nrows / 128), 1), st, D, P, y, maxkey)));
    }
    return FW_OK;
  }
  int pair_bulk(cudaStream_t st, int Pp, bool last, bool pdl = false) {
    const int a = 2 * Pp, kb = a * BS, w = (last ? 2 : 4) * BS;
    TileArgs t = tile_args(ld, bpair(Pp), ld, kb, 2 * BS, a, nrows, n_pad);
    put(t, 0, Strip{0, 0, lrow(a), lrow(a) + w, kb, kb + w, 0});
    return launch_tile<T, 128, 128, MODE>(dim3((unsigned)(n_pad / 128), (unsigned)(nrows / 128), 1), st, D, P,
                                          t, maxkey, pdl);
  }
  // The same schedule with each bulk launch (after the first) programmatically serialized with
  // the previous one: its CTAs take the SMs the previous launch's last wave frees and run their
  // main loops (which read only blocks a, b: final once the pivot stream is done) before they
  // wait for that launch in the epilogue. Only disable-timing events sit between two bulk
  // launches in st (a timing event there serializes them); the solve is timed from the first
  // bulk launch to the last (e.ev[3 P0], e.ev[3 (NP-1) + 2]).
  int run_pairs_pdl(cudaStream_t st, const Events &e, int P0, int NP) {
    cudaStream_t side = c.side;
    TRY(ensure_xev(c, (size_t)NP));
    TRY(pair_pivot(st, P0));
    if (e.timing) CU(cudaEventRecord(e.ev[3 * P0], st));
    for (int Pp = P0; Pp < NP; ++Pp) {
      Nvtx nv("pair");
      const bool last = Pp + 1 == NP;
      if (!last) {
        CU(cudaEventRecord(c.xev[Pp], st));            // the previous bulk launch is done
        CU(cudaStreamWaitEvent(side, c.xev[Pp], 0));
        if (e.timing) CU(cudaEventRecord(e.sync[2 * Pp], side));
        TRY(pair_prio(side, Pp));
        TRY(pair_pivot(side, Pp + 1));
        CU(cudaEventRecord(e.sync[2 * Pp + 1], side));
      }
      TRY(pair_bulk(st, Pp, last, Pp > P0));
      if (!last) CU(cudaStreamWaitEvent(st, e.sync[2 * Pp + 1], 0));
    }
    if (e.timing) CU(cudaEventRecord(e.ev[3 * (NP - 1) + 2], st));
    c.last_pdl = true;
    return FW_OK;
  }

  // Rounds [K0, K1) (K0, K1 even, blocks K0..K1-1 inside these rows) in pairs.
  int run_pairs(cudaStream_t st, const Events &e, int K0 = 0, int K1 = -1) {
    if (K1 < 0) K1 = R;
    const int P0 = K0 / 2, NP = K1 / 2;
    if (P0 >= NP) return FW_OK;
    cudaStream_t side = c.side;
    const bool overlap = c.pair_order;
    if (overlap && c.pair_pdl) return run_pairs_pdl(st, e, P0, NP);
    TRY(pair_pivot(st, P0));
    for (int Pp = P0; Pp < NP; ++Pp) {
      Nvtx nv("pair");
      const bool last = Pp + 1 == NP;
      if (e.timing) CU(cudaEventRecord(e.ev[3 * Pp], st));        // the pair's phase-3 work starts
      if (!last && overlap) {
        // the next pair's strips on the (high-priority) pivot stream, concurrent with the bulk
        // launch: their CTAs are dispatched first and the bulk fills the SMs behind their tail
        CU(cudaEventRecord(e.sync[2 * Pp], st));                  // the previous bulk launch is done
        CU(cudaStreamWaitEvent(side, e.sync[2 * Pp], 0));
        TRY(pair_prio(side, Pp));
        TRY(pair_pivot(side, Pp + 1));
        CU(cudaEventRecord(e.sync[2 * Pp + 1], side));
        TRY(pair_bulk(st, Pp, last));
      } else {
        if (!last) {
          TRY(pair_prio(st, Pp));
          CU(cudaEventRecord(e.sync[2 * Pp], st));
          CU(cudaStreamWaitEvent(side, e.sync[2 * Pp], 0));
          TRY(pair_pivot(side, Pp + 1));
          CU(cudaEventRecord(e.sync[2 * Pp + 1], side));
        }
        TRY(pair_bulk(st, Pp, last));
      }
      if (e.timing) CU(cudaEventRecord(e.ev[3 * Pp + 2], st));    // ... and ends
      if (!last) CU(cudaStreamWaitEvent(st, e.sync[2 * Pp + 1], 0));
    }
    return FW_OK;
  }

  // Rounds [K0, K1) of these rows (default: all). A row range of the host pipeline runs
  // its rounds in several calls; every round's pivot strip must have completed that round.
  int run(cudaStream_t st, const Events &e, bool lookahead, int K0 = 0, int K1 = -1) {
    cudaEvent_t *ev = e.ev;
    if (K1 < 0) K1 = R;
    if (K0 >= K1) return FW_OK;
    if (!lookahead || BS != 128 || K1 - K0 < 2) {
      for (int K = K0; K < K1; ++K) {
        TRY(phase1(st, K));
        if (e.timing) CU(cudaEventRecord(ev[3 * K], st));
        TRY(pivot_rest(st, K));
        if (e.timing) CU(cudaEventRecord(ev[3 * K + 1], st));
        TRY(phase3_full(st, K));
        if (e.timing) CU(cudaEventRecord(ev[3 * K + 2], st));
      }
      return FW_OK;
    }
    if (world == 1 && c.pair_pdl) return run_pdl(st, e, K0, K1);
    cudaStream_t side = c.side;
    TRY(phase1(st, K0));
    if (e.timing) CU(cudaEventRecord(ev[3 * K0], st));
    TRY(pivot_rest(st, K0));
    if (e.timing) CU(cudaEventRecord(ev[3 * K0 + 1], st));
    CU(cudaEventRecord(e.sync[2 * K0], st));
    CU(cudaStreamWaitEvent(side, e.sync[2 * K0], 0));   // the pivot stream follows round K0's pivot
    for (int K = K0; K < K1; ++K) {
      Nvtx nv("round");
      if (K + 1 < K1) {
        int nprio = 0;
        TRY(phase3_ordered(st, K, done + K, &nprio));
        if (e.timing) CU(cudaEventRecord(ev[3 * K + 2], st));
        // pivot stream: wait for the look-ahead tiles of round K, then round K+1's pivot
        TRY(wait_count(side, K, nprio));
        if (e.timing) CU(cudaEventRecord(e.sync[2 * K + 2], side));
        TRY(phase1(side, K + 1));
        if (e.timing) CU(cudaEventRecord(ev[3 * (K + 1)], side));
        TRY(pivot_rest(side, K + 1));
        if (e.timing) CU(cudaEventRecord(ev[3 * (K + 1) + 1], side));
        CU(cudaEventRecord(e.sync[2 * K + 1], side));
        CU(cudaStreamWaitEvent(st, e.sync[2 * K + 1], 0));
      } else {
        TRY(phase3_full(st, K));
        if (e.timing) CU(cudaEventRecord(ev[3 * K + 2], st));
      }
    }
    return FW_OK;
  }

  // The look-ahead schedule (one GPU) with each ordered launch after the first programmatically
  // serialized with the previous one (as run_pairs_pdl): launch K's main loop (column block K,
  // row K: look-ahead tiles of launch K-1, final once the pivot stream's event fired) overlaps
  // launch K-1's last wave; its epilogue waits for launch K-1. The pivot stream now also waits
  // for launch K-1 to complete (xev[K]) before round K+1's phases, which rewrite tiles of row
  // and column K+1 that launch K-1 may still be writing. Main-stream events between ordered
  // launches are disable-timing (a timing record would serialize them).
  int run_pdl(cudaStream_t st, const Events &e, int K0, int K1) {
    cudaEvent_t *ev = e.ev;
    cudaStream_t side = c.side;
    TRY(ensure_xev(c, (size_t)K1));
    TRY(phase1(st, K0));
    if (e.timing) CU(cudaEventRecord(ev[3 * K0], st));
    TRY(pivot_rest(st, K0));
    if (e.timing) CU(cudaEventRecord(ev[3 * K0 + 1], st));
    for (int K = K0; K < K1; ++K) {
      Nvtx nv("round");
      if (K + 1 < K1) {
        CU(cudaEventRecord(c.xev[K], st));           // launch K-1 (and round K's pivot) complete
        int nprio = 0;
        TRY(phase3_ordered(st, K, done + K, &nprio, K > K0));
        CU(cudaStreamWaitEvent(side, c.xev[K], 0));
        TRY(wait_count(side, K, nprio));
        if (e.timing) CU(cudaEventRecord(e.sync[2 * K + 2], side));
        TRY(phase1(side, K + 1));
        if (e.timing) CU(cudaEventRecord(ev[3 * (K + 1)], side));
        TRY(pivot_rest(side, K + 1));
        if (e.timing) CU(cudaEventRecord(ev[3 * (K + 1) + 1], side));
        CU(cudaEventRecord(e.sync[2 * K + 1], side));
        CU(cudaStreamWaitEvent(st, e.sync[2 * K + 1], 0));
      } else {
        TRY(phase3_full(st, K, K > K0));
      }
    }
    if (e.timing) CU(cudaEventRecord(ev[3 * (K1 - 1) + 2], st));
    c.last_pdl = true;
    return FW_OK;
  }

  // pivot phases after phase 1: strips and (multi-GPU) the broadcast
  int pivot_rest(cudaStream_t st, int K) { return phase2(st, K, true, true); }
};

// ---- the multi-rank round driver (SURVEY §8 e) --------------------------------------------
// The ranks of a block-row partition that this host thread drives: ONE (this process's rank of
// an NCCL communicator, any world size) or ALL W (the loopback transport: every rank emulated on
// this GPU). Every rank has a main stream and a high-priority look-ahead stream with run()'s
// event structure — the look-ahead tiles first in an ordered phase-3 launch on the main stream,
// a wait_count_kernel gate and the next round's pivot phases on the look-ahead stream, the main
// stream waiting for them — and the pivot rows go from their owner to every other rank through
// ncclBroadcast (NCCL) or, in the loopback, a device copy per receiver with a collective's
// completion semantics: each receiver's copy is ordered on ITS stream after the owner's strips,
// and the owner's stream continues only after every receiver's copy. So the schedule the NCCL
// ranks run is exactly the one the loopback tests run on one GPU, concurrently: the cross-stream
// reuse of the two strip buffers and of the owner's pivot rows is exercised — on G GPUs it is
// safe only through the chain "look-ahead tiles of launch K done => launch K started => launch
// K-1, the last reader of strip[(K+1) & 1], complete". Every wait is for work that waits on
// nothing (wait_count_kernel is one thread and bounded), so the emulation cannot deadlock.
//
// Pairs (keyed / plain solves, BS = 128, R even, every rank's rows aligned to 256; DESIGN.md
// §4.9, §9): the owner of blocks a, b = 2P, 2P+1 runs the one-GPU pair pivot on its rows, the
// 256 rows a, b go out in ONE broadcast, the other ranks bring their columns a, b through both
// rounds (pair_cols), and every rank relaxes its other tiles through 256 k in one bulk launch;
// the next pair's strips (pair_prio) and pivot path run on the look-ahead streams under it.
int ensure_lb(Ctx &c, int W) {
  int lo = 0, hi = 0;
  CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  while ((int)c.lb_st.size() < 2 * W) {
    cudaStream_t q;
    CU(cudaStreamCreateWithPriority(&q, cudaStreamNonBlocking, c.lb_st.size() % 2 ? hi : lo));
    c.lb_st.push_back(q);
  }
  while ((int)c.lb_ev.size() < 1 + 3 * W) {
    cudaEvent_t e;
    CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c.lb_ev.push_back(e);
  }
  return FW_OK;
}

// every rank's rows start on a 256-row boundary (pairs of blocks never straddle two ranks)
bool pairs_aligned(int64_t n, int world) {
  for (int r = 0; r < world; ++r) {
    int64_t r0, nr;
    partition(n, world, r, &r0, &nr);
    if (r0 % 256) return false;
  }
  return true;
}

template <typename T, int MODE>
struct Team {
  Ctx &c;
  std::vector<Rounds<T, MODE>> &rk;
  bool nccl;                   // one local rank of an NCCL communicator; else the loopback
  const Events &e;             // timing events of local rank 0 (NCCL only)
  cudaStream_t st;             // the solve's stream
  cudaStream_t *ms = nullptr;  // ms[2r]: local rank r's main stream, ms[2r + 1]: its look-ahead stream
  cudaStream_t pair_nccl[2] = {nullptr, nullptr};
  cudaEvent_t *ev = nullptr;   // [0] root, [1 + r] receive, [1 + W + r], [1 + 2W + r] follow
  int W() const { return (int)rk.size(); }
  cudaStream_t q(int r, int side) const { return ms[2 * r + side]; }
  int BS() const { return rk[0].BS; }

  int setup() {
    if (nccl) {
      pair_nccl[0] = st;
      pair_nccl[1] = c.side;
      ms = pair_nccl;
      TRY(ensure_lb(c, 1));        // events only
      ev = c.lb_ev.data();
      return FW_OK;
    }
    TRY(ensure_lb(c, W()));
    ms = c.lb_st.data();
    ev = c.lb_ev.data();
    CU(cudaEventRecord(ev[0], st));                    // fork: every rank's streams follow st
    for (int r = 0; r < 2 * W(); ++r) CU(cudaStreamWaitEvent(ms[r], ev[0], 0));
    return FW_OK;
  }
  int join() {
    if (nccl) return FW_OK;       // the main stream is st
    for (int r = 0; r < 2 * W(); ++r) TRY(follow(st, ms[r], ev[1 + W() + r / 2]));
    return FW_OK;
  }
  int follow(cudaStream_t waiter, cudaStream_t src, cudaEvent_t x) {
    CU(cudaEventRecord(x, src));
    CU(cudaStreamWaitEvent(waiter, x, 0));
    return FW_OK;
  }
  void mark(cudaEvent_t x, int r, int side) {   // a timing event of local rank 0
    if (e.timing && r == 0) cudaEventRecord(x, q(0, side));
  }

  // rows [K*BS, (K+nb)*BS) from their owner into strip[slot] of every other rank
  int bcast(int K, int nb, int slot, int side) {
    Nvtx nv("broadcast");
    Rounds<T, MODE> &x0 = rk[0];
    const int64_t n_pad = x0.n_pad;
    const size_t count = (size_t)nb * BS() * (size_t)n_pad;
    if (nccl) {
      void *buf = x0.owns(K) ? (void *)(x0.D + (int64_t)x0.lrow(K) * x0.ld) : (void *)x0.strip[slot];
      NCC(c, g_nccl.Broadcast(buf, buf, count, std::is_integral<T>::value ? ncclInt32 : ncclFloat32,
                              owner_of(n_pad, x0.world, (int64_t)K * BS()), c.comm, q(0, side)));
      ++g_bcasts;
      g_bcast_bytes += (double)count * sizeof(T);
      return FW_OK;
    }
    const int o = owner_of(n_pad, W(), (int64_t)K * BS());
    CU(cudaEventRecord(ev[0], q(o, side)));
    const T *src = rk[o].D + (int64_t)rk[o].lrow(K) * rk[o].ld;
    for (int r = 0; r < W(); ++r) {
      if (r == o) continue;
      CU(cudaStreamWaitEvent(q(r, side), ev[0], 0));
      CU(cudaMemcpy2DAsync(rk[r].strip[slot], n_pad * sizeof(T), src, rk[o].ld * sizeof(T), n_pad * sizeof(T),
                           (size_t)nb * BS(), cudaMemcpyDeviceToDevice, q(r, side)));
      CU(cudaEventRecord(ev[1 + r], q(r, side)));
    }
    for (int r = 0; r < W(); ++r)
      if (r != o) CU(cudaStreamWaitEvent(q(o, side), ev[1 + r], 0));
    return FW_OK;
  }

  // round K's pivot phases: phase 1 and the row strip on the owner, the broadcast, every rank's
  // column strip (phase1 / the row strip are no-ops on ranks that do not own block K)
  int pivot(int K, int side) {
    Nvtx nv("pivot phases");
    for (int r = 0; r < W(); ++r) {
      TRY(rk[r].phase1(q(r, side), K));
      mark(e.ev[3 * K], r, side);
      TRY(rk[r].phase2(q(r, side), K, true, false));
    }
    TRY(bcast(K, 1, K & 1, side));
    for (int r = 0; r < W(); ++r) {
      TRY(rk[r].phase2(q(r, side), K, false, true));
      mark(e.ev[3 * K + 1], r, side);
    }
    return FW_OK;
  }

  int run_rounds(bool lookahead) {
    Rounds<T, MODE> &x0 = rk[0];
    const int R = x0.R;
    if (!lookahead || BS() != 128 || R < 2) {
      for (int K = 0; K < R; ++K) {
        TRY(pivot(K, 0));
        for (int r = 0; r < W(); ++r) {
          TRY(rk[r].phase3_full(q(r, 0), K));
          mark(e.ev[3 * K + 2], r, 0);
        }
      }
      return FW_OK;
    }
    TRY(pivot(0, 0));
    for (int r = 0; r < W(); ++r) TRY(follow(q(r, 1), q(r, 0), ev[1 + W() + r]));   // side follows round 0's pivot
    for (int K = 0; K < R; ++K) {
      if (K + 1 < R) {
        Nvtx nv("round");
        for (int r = 0; r < W(); ++r) {
          int nprio = 0;
          TRY(rk[r].phase3_ordered(q(r, 0), K, rk[r].done + K, &nprio));
          mark(e.ev[3 * K + 2], r, 0);
          TRY(rk[r].wait_count(q(r, 1), K, nprio));
          mark(e.sync[2 * K + 2], r, 1);
        }
        TRY(pivot(K + 1, 1));
        for (int r = 0; r < W(); ++r) TRY(follow(q(r, 0), q(r, 1), ev[1 + 2 * W() + r]));
      } else {
        for (int r = 0; r < W(); ++r) {
          TRY(rk[r].phase3_full(q(r, 0), K));
          mark(e.ev[3 * K + 2], r, 0);
        }
      }
    }
    return FW_OK;
  }

  // pair Pp's pivot path: the owner's pair pivot on its rows, ONE broadcast of rows a, b, the
  // other ranks' columns a, b
  int pair_pivot(int Pp, int side) {
    Nvtx nv("pair pivot");
    const int a = 2 * Pp;
    for (int r = 0; r < W(); ++r)
      if (rk[r].owns(a)) TRY(rk[r].pair_pivot(q(r, side), Pp));
    TRY(bcast(a, 2, Pp & 1, side));
    for (int r = 0; r < W(); ++r)
      if (!rk[r].owns(a)) TRY(rk[r].pair_cols(q(r, side), Pp));
    return FW_OK;
  }

  int run_pairs() {
    const int NP = rk[0].R / 2;
    TRY(pair_pivot(0, 0));
    for (int Pp = 0; Pp < NP; ++Pp) {
      Nvtx nv("pair");
      const bool last = Pp + 1 == NP;
      for (int r = 0; r < W(); ++r) mark(e.ev[3 * Pp], r, 0);           // the pair's phase-3 work starts
      if (!last) {
        for (int r = 0; r < W(); ++r) {
          TRY(follow(q(r, 1), q(r, 0), ev[1 + W() + r]));               // the previous bulk launch is done
          mark(e.sync[2 * Pp], r, 1);
          TRY(rk[r].pair_prio(q(r, 1), Pp));
        }
        TRY(pair_pivot(Pp + 1, 1));
        for (int r = 0; r < W(); ++r) {
          mark(e.sync[2 * Pp + 1], r, 1);
          CU(cudaEventRecord(ev[1 + 2 * W() + r], q(r, 1)));
        }
      }
      for (int r = 0; r < W(); ++r) {
        TRY(rk[r].pair_bulk(q(r, 0), Pp, last));
        mark(e.ev[3 * Pp + 2], r, 0);
        if (!last) CU(cudaStreamWaitEvent(q(r, 0), ev[1 + 2 * W() + r], 0));
      }
    }
    return FW_OK;
  }
};

template <typename T, int MODE>
int run_team(Ctx &c, std::vector<Rounds<T, MODE>> &rk, bool nccl, cudaStream_t st, const Events &e, bool la,
             bool pairs) {
  Team<T, MODE> t{c, rk, nccl, e, st};
  TRY(t.setup());
  TRY(pairs ? t.run_pairs() : t.run_rounds(la));
  return t.join();
}


// ---- the solve ---------------------------------------------------------------------------
enum Transport { T_LOCAL = 0, T_NCCL = 1, T_LOOPBACK = 2 };

// One rank's part of a solve: the caller's rows and where they are solved.
template <typename T>
struct Part {
  T *src;            // caller's rows [row0, row0 + nsrc) of the n x n matrix, pitch ld_src
  int64_t ld_src;
  int32_t *next;     // same rows of P, pitch ld_next, or nullptr
  int64_t ld_next;
  int rank;
  int64_t row0, nrows, nsrc;
  T *D = nullptr;    // padded working rows (nrows x n_pad, pitch ld)
  int32_t *P = nullptr;
  int64_t ld = 0;
  bool inplace = false;
  T *strip[2] = {nullptr, nullptr};
  T *backup = nullptr;
};

template <typename R> int *maxkey_of(std::vector<R> &rk) { return rk[0].maxkey; }

template <typename T, int MODE>
int launch_persistent(Ctx &c, std::vector<RankView> &views, int64_t ld, int64_t n_pad, int *maxkey,
                      cudaStream_t st, const Events &e, int self = -1,
                      const std::function<int()> &barrier = nullptr);

// The whole solve as one persistent launch (fw_persist.cuh): one GPU, all rows,
// BS = 128. Auto: round-tag solves (real-valued data, one round per pass). Keyed and
// distance-only solves keep the two-rounds-per-pass schedule (§4.9), whose 256-deep bulk
// launches the persistent one-round items do not match.
bool use_persistent(const Ctx &c, int mode, int tr, int BS, int64_t n_pad, int64_t row0, int64_t nrows) {
  if (tr != T_LOCAL || BS != 128 || row0 != 0 || nrows != n_pad || c.persistent == 0) return false;
  if (c.persistent == 1) return true;
  // auto: round-tag solves up to n = 4096, where the stream-ordered rounds are bound by the
  // per-round pivot path (C2); above, its tiles run ~8% slower than the stream kernel's
  //
  return mode == MODE_TAG && n_pad >= 4 * 128 && n_pad <= 4096;
}

// Item table of a multi-rank persistent solve (fw_persist.cuh): per round K a segment
//   A  prio(K): every rank's round-K tiles of row K+1 (its owner; (K+1, K+1) first) and of
//      column K+1 (rows outside K, K+1)
//   B  P1(K+1) on the owner of block K+1
//   C  the first `gap` other phase-3 tiles of round K, per rank
//   D  P2(K+1): the owner's row K+1 tiles, then every rank's column K+1 tiles
//   E  the remaining phase-3 tiles of round K
// (preamble: P1(0), P2(0); the last segment: round T-1's phase-3 tiles). Every item depends only
// on items earlier in this order (same argument as the one-rank order; cross-rank: a rank's
// phase-2 column tiles and phase-3 tiles read published pivot tiles from segments B / D or
// earlier). self >= 0: that rank's items only (a team: one grid per GPU) — each GPU's sequence
// is then a subsequence of the global order, whose cross-GPU dependencies point only to earlier
// segments or to the owner's phase B / D items, which depend on nothing later: no cycle.
void persist_items(int T, int world, const std::vector<int> &t0, const std::vector<int> &t1, int self, int gap,
                   std::vector<unsigned> *out) {
  std::vector<unsigned> &v = *out;
  v.clear();
  auto owner = [&](int K) {
    int o = 0;
    for (int q = 1; q < world; ++q)
      if (K >= t0[q]) o = q;
    return o;
  };
  auto take = [&](int r) { return self < 0 || r == self; };
  auto tile = [&](int r, int K, int I, int J) {
    if (take(r)) v.push_back(pack_item(r, IT_TILE, K, I, J));
  };
  const int o0 = owner(0);
  if (take(o0)) v.push_back(pack_item(o0, IT_P1, 0, 0, 0));
  for (int J = 1; J < T; ++J) tile(o0, 0, 0, J);
  for (int r = 0; r < world; ++r)
    for (int I = t0[r]; I < t1[r]; ++I)
      if (I != 0) tile(r, 0, I, 0);
  for (int K = 0; K < T; ++K) {
    const int N = K + 1;
    if (N == T) {
      for (int r = 0; r < world; ++r)
        for (int I = t0[r]; I < t1[r]; ++I)
          if (I != K)
            for (int J = 0; J < T; ++J)
              if (J != K) tile(r, K, I, J);
      break;
    }
    const int oN = owner(N);
    tile(oN, K, N, N);                                                  // A
    for (int J = 0; J < T; ++J)
      if (J != K && J != N) tile(oN, K, N, J);
    for (int r = 0; r < world; ++r)
      for (int I = t0[r]; I < t1[r]; ++I)
        if (I != K && I != N) tile(r, K, I, N);
    if (take(oN)) v.push_back(pack_item(oN, IT_P1, N, N, N));          // B
    // rest(K): row and column M = K+2 first ((M, M) first; the next round's prio tiles wait for
    // them, persist_rest_ij), then row-major — per rank, its rows only
    std::vector<std::vector<unsigned>> rest(world);
    const int M = K + 2;
    for (int r = 0; r < world; ++r) {
      auto push = [&](int I, int J) { rest[r].push_back(pack_item(r, IT_TILE, K, I, J)); };
      const bool ownM = M < T && M >= t0[r] && M < t1[r];
      if (ownM) {
        push(M, M);
        for (int J = 0; J < T; ++J)
          if (J != K && J != N && J != M) push(M, J);
      }
      if (M < T)
        for (int I = t0[r]; I < t1[r]; ++I)
          if (I != K && I != N && I != M) push(I, M);
      for (int I = t0[r]; I < t1[r]; ++I)
        if (I != K && I != N && (M >= T || I != M))
          for (int J = 0; J < T; ++J)
            if (J != K && J != N && (M >= T || J != M)) push(I, J);
    }
    for (int r = 0; r < world; ++r)                                      // C
      if (take(r))
        for (size_t q = 0; q < rest[r].size() && (int)q < gap; ++q) v.push_back(rest[r][q]);
    for (int J = 0; J < T; ++J)                                          // D
      if (J != N) tile(oN, N, N, J);
    for (int r = 0; r < world; ++r)
      for (int I = t0[r]; I < t1[r]; ++I)
        if (I != N) tile(r, N, I, N);
    for (int r = 0; r < world; ++r)                                      // E
      if (take(r))
        for (size_t q = gap; q < rest[r].size(); ++q) v.push_back(rest[r][q]);
  }
}

// One persistent launch over the ranks of `views` (world = 1: all rows of one GPU, items
// decoded arithmetically; world > 1: a loopback partition emulated in ONE grid — the guide's way
// to test ranks that wait on one another on one GPU — with the item table and the rings).
// self >= 0: this process runs rank `self` of a communicator (its items only); the views' ring /
// pub pointers (peers' mapped through CUDA IPC) and the zeroing of its pub flags are the
// caller's, and `barrier` runs between the zeroing and the launch.
template <typename T, int MODE>
int launch_persistent(Ctx &c, std::vector<RankView> &views, int64_t ld, int64_t n_pad, int *maxkey,
                      cudaStream_t st, const Events &e, int self, const std::function<int()> &barrier) {
  const int Tn = (int)(n_pad / 128), W = (int)views.size();
  if (W > kMaxRanks) return fail(FW_EINVAL, "persistent solve: at most %d ranks", kMaxRanks);
  auto kern = fw_persistent_kernel<T, MODE>;
  constexpr int bytes = TileShape<128, 128>::kBytes;
  TRY(smem_attr((const void *)kern, bytes));
  int dev = 0, sms = 0, per_sm = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, bytes));
  if (per_sm < 1) return fail(FW_ECUDA, "fw_persistent_kernel does not fit on an SM");
  const bool p1_lone = W == 1 && per_sm >= 2 && c.persist_p1_lone != 0;
  const int grid = per_sm * sms - (p1_lone ? 1 : 0);   // p1_lone: one SM keeps a single CTA
  // counters: per rank its tiles' round counters, and (W > 1) pub flags of its ring; then the
  // 64-bit work counter, 256-B aligned
  size_t off = 0;
  std::vector<size_t> ver_off(W), pub_off(W);
  for (int r = 0; r < W; ++r) {
    ver_off[r] = off;
    off += ((size_t)(views[r].t1 - views[r].t0) * Tn * sizeof(int) + 255) / 256 * 256;
    pub_off[r] = off;
    if (W > 1 && self < 0) off += ((size_t)Tn * Tn * sizeof(int) + 255) / 256 * 256;
  }
  const size_t qcnt_off = off;   // one GPU: per-tile count of finished quarter items
  off += W == 1 ? ((size_t)Tn * Tn * sizeof(int) + 255) / 256 * 256 : 0;
  const size_t next_off = off;
  off += 256;
  const size_t smcnt_off = off;   // p1_lone: per-SM CTA counts + the start barrier count
  off += ((size_t)(sms + 1) * sizeof(int) + 255) / 256 * 256;
  const int gap = c.persist_gap >= 0 ? c.persist_gap : 2 * grid;   // C2: 600 best of 300-900
  std::vector<unsigned> items;
  if (W > 1) {
    std::vector<int> t0(W), t1(W);
    for (int r = 0; r < W; ++r) t0[r] = views[r].t0, t1[r] = views[r].t1;
    persist_items(Tn, W, t0, t1, self, gap, &items);
  }
  const size_t items_off = off;
  off += (items.size() * sizeof(unsigned) + 255) / 256 * 256;
  // FW_PERSIST_TRACE=path (development): every item's {taken, operands ready, done} times and
  // its SM / CTA, written to `path` after the launch (tools/persist_trace.py reads it)
  const char *trace_path = getenv("FW_PERSIST_TRACE");
  // quarters shorten the per-round pivot chain, which bounds small solves (n = 2048: 2.07 -> 1.50
  // ms, n = 3072: 3.37 -> 2.78 ms with every prio / P2 tile quartered)
  // auto: every chain tile in quarters up to T = 16 (n = 1024: 0.75 vs 0.82 ms, n = 2048: 1.54 vs
  // 1.56), only the three chain tiles per round from T = 24 on (n = 3072: 2.65 vs 2.70, C2: 5.33
  // vs 5.43 ms with none; profiles/r02c_persist_quarters_ab.jsonl)
  const int qmode = W != 1 ? 0 : c.persist_quarters < 0 ? (Tn < 20 ? 1 : 2) : c.persist_quarters;
  const int Qt = qmode == 1 ? 4 : 1;
  const long long total_items = W > 1 ? (long long)items.size()
                                : qmode == 2 ? persist_total_crit(Tn)
                                             : 1 + (long long)Qt * 2 * (Tn - 1) +
                                                   (long long)Tn * ((long long)Tn * Tn + (Qt - 1) * (4LL * Tn - 5));
  const size_t trace_off = off;
  if (trace_path && *trace_path) off += (size_t)(total_items + Tn) * 64;   // + the dedicated P1 CTA's
  TRY(c.ws_ver.ensure(off));
  char *base = static_cast<char *>(c.ws_ver.p);
  CU(cudaMemsetAsync(base, 0, items_off, st));
  if (trace_path && *trace_path) CU(cudaMemsetAsync(base + trace_off, 0, (size_t)(total_items + Tn) * 64, st));
  if (!items.empty())
    CU(cudaMemcpyAsync(base + items_off, items.data(), items.size() * sizeof(unsigned), cudaMemcpyHostToDevice, st));
  PersistArgs a{};
  a.ld = ld;
  a.ldr = n_pad;
  a.T = Tn;
  // P1(K+1) takes about one tile wait + 1.6 tile times; the P2(K+1) items go in after roughly that
  // many grid-waves of round K's phase-3 tiles, so they rarely wait
  a.gap = gap;
  a.world = W;
  a.items = items.empty() ? nullptr : reinterpret_cast<const unsigned *>(base + items_off);
  a.next = reinterpret_cast<unsigned long long *>(base + next_off);
  a.maxkey = maxkey;
  a.flags = maxkey - 2;
  a.quarters = qmode;
  a.qcnt = reinterpret_cast<int *>(base + qcnt_off);
  a.p1_lone = p1_lone ? 1 : 0;
  a.stage_old = c.persist_stage_old != 0 ? 1 : 0;
  a.smcnt = reinterpret_cast<int *>(base + smcnt_off);
  a.nsm = sms;
  a.total = total_items;
  a.timeout_ns = 20ull * 1000 * 1000 * 1000;
  a.trace = trace_path && *trace_path ? reinterpret_cast<unsigned long long *>(base + trace_off) : nullptr;
  a.sync_relaxed = c.persist_relaxed;
  a.p1_blocked = g_p1_blocked != 0;
  for (int r = 0; r < W; ++r) {
    a.rk[r] = views[r];
    a.rk[r].ver = reinterpret_cast<int *>(base + ver_off[r]);
    if (self < 0) a.rk[r].pub = W > 1 ? reinterpret_cast<int *>(base + pub_off[r]) : nullptr;
  }
  if (barrier) TRY(barrier());
  Nvtx nv("persistent solve");
  if (e.timing) CU(cudaEventRecord(e.ev[0], st));
  kern<<<grid, kThreads, bytes, st>>>(a);
  ++g_launches;
  CU(cudaGetLastError());
  if (e.timing) CU(cudaEventRecord(e.ev[2], st));
  if (a.trace) {
    std::vector<unsigned long long> h((size_t)(total_items + Tn) * 8);
    CU(cudaMemcpyAsync(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (FILE *f = fopen(trace_path, "wb")) {
      const long long hdr[8] = {0x46575453, Tn, W, total_items, a.quarters, a.gap, grid, self};
      fwrite(hdr, sizeof hdr, 1, f);
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
  }
  return FW_OK;
}

template <typename T, int MODE>
int run_persistent(Ctx &c, T *D, int32_t *P, int64_t ld, int64_t n_pad, int *maxkey, cudaStream_t st,
                   const Events &e) {
  std::vector<RankView> v(1);
  v[0] = RankView{D, P, nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0, (int)(n_pad / 128)};
  return launch_persistent<T, MODE>(c, v, ld, n_pad, maxkey, st, e);
}

// One rank of a communicator (one process per GPU) as a persistent grid with the fused publish
// (opt-in: fw_set_option("persistent", 1)): every rank allocates its pivot-row
// ring + pub flags, the CUDA IPC handles are all-gathered over NCCL and mapped (NVLink peer
// access), each rank zeroes its own flags, an NCCL all-reduce is the barrier before the launch,
// and the owner of each pivot-row tile stores it straight into the peers' rings (P2P stores over
// NVLink) with a system-scope release flag — no ncclBroadcast in the rounds. The all-reduces of
// the next solve's validation order its zeroing after every peer's kernel. NOT run on hardware:
// the gpurun boxes have one GPU (the protocol is tested by the loopback grid above).
// ---- NVLS: the pivot-row rings of a communicator as one multicast object --------
// With NVSwitch multicast (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED) every rank's ring is physical
// memory bound to ONE multicast object, so the fused publish stores each final pivot-row tile once
// (multimem.st) and the switch replicates it into every ring — instead of G-1 peer copies through
// the owner's links. Set up collectively over the communicator: rank 0 creates the
// object and exports a fabric handle, the others import it, every rank adds its device, binds its
// ring memory and maps it twice (unicast: its own ring; multicast: the publish address). Any
// failure on any rank (no multicast support, no fabric handles — e.g. a pool that shows each
// process one GPU) drops every rank back to the IPC peer rings; the driver API is reached through
// cudaGetDriverEntryPoint (no link-time libcuda dependency).
struct CuApi {
  bool tried = false, ok = false;
  decltype(&cuDeviceGetAttribute) DeviceGetAttribute;
  decltype(&cuDeviceGet) DeviceGet;
  decltype(&cuMulticastGetGranularity) MulticastGetGranularity;
  decltype(&cuMulticastCreate) MulticastCreate;
  decltype(&cuMulticastAddDevice) MulticastAddDevice;
  decltype(&cuMulticastBindMem) MulticastBindMem;
  decltype(&cuMulticastUnbind) MulticastUnbind;
  decltype(&cuMemExportToShareableHandle) MemExportToShareableHandle;
  decltype(&cuMemImportFromShareableHandle) MemImportFromShareableHandle;
  decltype(&cuMemCreate) MemCreate;
  decltype(&cuMemRelease) MemRelease;
  decltype(&cuMemAddressReserve) MemAddressReserve;
  decltype(&cuMemAddressFree) MemAddressFree;
  decltype(&cuMemMap) MemMap;
  decltype(&cuMemUnmap) MemUnmap;
  decltype(&cuMemSetAccess) MemSetAccess;
} g_cu;

bool load_cu() {
  if (g_cu.tried) return g_cu.ok;
  g_cu.tried = true;
  bool ok = true;
  auto get = [&](const char *name, auto &fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      ok = false;
      return;
    }
    fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(p);
  };
  get("cuDeviceGetAttribute", g_cu.DeviceGetAttribute);
  get("cuDeviceGet", g_cu.DeviceGet);
  get("cuMulticastGetGranularity", g_cu.MulticastGetGranularity);
  get("cuMulticastCreate", g_cu.MulticastCreate);
  get("cuMulticastAddDevice", g_cu.MulticastAddDevice);
  get("cuMulticastBindMem", g_cu.MulticastBindMem);
  get("cuMulticastUnbind", g_cu.MulticastUnbind);
  get("cuMemExportToShareableHandle", g_cu.MemExportToShareableHandle);
  get("cuMemImportFromShareableHandle", g_cu.MemImportFromShareableHandle);
  get("cuMemCreate", g_cu.MemCreate);
  get("cuMemRelease", g_cu.MemRelease);
  get("cuMemAddressReserve", g_cu.MemAddressReserve);
  get("cuMemAddressFree", g_cu.MemAddressFree);
  get("cuMemMap", g_cu.MemMap);
  get("cuMemUnmap", g_cu.MemUnmap);
  get("cuMemSetAccess", g_cu.MemSetAccess);
  g_cu.ok = ok;
  return ok;
}

void nvls_release(Ctx &c) {
  Ctx::Nvls &v = c.nvls;
  if (!g_cu.ok) return;
  if (v.mcva) g_cu.MemUnmap(v.mcva, v.size), g_cu.MemAddressFree(v.mcva, v.size);
  if (v.uc) g_cu.MemUnmap(v.uc, v.size), g_cu.MemAddressFree(v.uc, v.size);
  CUdevice dev;
  if (v.mc && v.mem && g_cu.DeviceGet(&dev, c.dev) == CUDA_SUCCESS) g_cu.MulticastUnbind(v.mc, dev, 0, v.size);
  if (v.mem) g_cu.MemRelease(v.mem);
  if (v.mc) g_cu.MemRelease(v.mc);
  v = Ctx::Nvls{};
}

// Collective: every rank of c.comm calls it with the same bytes. *ok = the multicast rings are
// usable on every rank (else all ranks use the IPC peer rings).
int nvls_setup(Ctx &c, size_t bytes, int W, int self, int *d_scratch, cudaStream_t st, bool *ok) {
  *ok = false;
  Ctx::Nvls &v = c.nvls;
  if (v.active && v.size >= bytes && v.world == W) {
    *ok = true;
    return FW_OK;
  }
  nvls_release(c);
  // one collective step: the minimum of every rank's status (1 = fine so far)
  auto agree = [&](int local, bool *all) -> int {
    CU(cudaMemcpyAsync(d_scratch, &local, sizeof local, cudaMemcpyHostToDevice, st));
    NCC(c, g_nccl.AllReduce(d_scratch, d_scratch, 1, ncclInt32, ncclMin, c.comm, st));
    int r = 0;
    CU(cudaMemcpyAsync(&r, d_scratch, sizeof r, cudaMemcpyDeviceToHost, st));
    TRY(sync_stream(c, st));
    *all = r == 1;
    return FW_OK;
  };
  bool all = false;
  CUdevice dev = 0;
  int mcs = 0;
  const int supported = c.nvls_opt != 0 && load_cu() && g_cu.DeviceGet(&dev, c.dev) == CUDA_SUCCESS &&
                        g_cu.DeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) == CUDA_SUCCESS &&
                        mcs == 1;
  TRY(agree(supported ? 1 : 0, &all));
  if (!all) return FW_OK;
  // rank 0: the multicast object and its fabric handle -> every rank
  struct Blob {
    int status;
    unsigned long long size;
    CUmemFabricHandle h;
  } blob{};
  if (self == 0) {
    CUmulticastObjectProp mp{};
    mp.numDevices = (unsigned)W;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
    mp.size = bytes;
    size_t gran = 0;
    blob.status = g_cu.MulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED) == CUDA_SUCCESS &&
                  gran > 0;
    if (blob.status) {
      mp.size = (bytes + gran - 1) / gran * gran;
      blob.size = mp.size;
      blob.status = g_cu.MulticastCreate(&v.mc, &mp) == CUDA_SUCCESS;
      if (blob.status)
        blob.status = g_cu.MemExportToShareableHandle(&blob.h, v.mc, CU_MEM_HANDLE_TYPE_FABRIC, 0) == CUDA_SUCCESS;
    }
  }
  TRY(c.ws_ipc.ensure(sizeof(Blob)));
  CU(cudaMemcpyAsync(c.ws_ipc.p, &blob, sizeof blob, cudaMemcpyHostToDevice, st));
  NCC(c, g_nccl.Broadcast(c.ws_ipc.p, c.ws_ipc.p, sizeof blob, ncclChar, 0, c.comm, st));
  CU(cudaMemcpyAsync(&blob, c.ws_ipc.p, sizeof blob, cudaMemcpyDeviceToHost, st));
  TRY(sync_stream(c, st));
  if (!blob.status) {
    nvls_release(c);
    return FW_OK;
  }
  v.size = (size_t)blob.size;
  int good = 1;
  if (self != 0) good = g_cu.MemImportFromShareableHandle(&v.mc, &blob.h, CU_MEM_HANDLE_TYPE_FABRIC) == CUDA_SUCCESS;
  if (good) good = g_cu.MulticastAddDevice(v.mc, dev) == CUDA_SUCCESS;
  TRY(agree(good, &all));   // every device is added before any memory is bound
  if (all) {
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = c.dev;
    CUmemAccessDesc ad{};
    ad.location = ap.location;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    good = g_cu.MemCreate(&v.mem, v.size, &ap, 0) == CUDA_SUCCESS;
    if (good) good = g_cu.MulticastBindMem(v.mc, 0, v.mem, 0, v.size, 0) == CUDA_SUCCESS;
    if (good) good = g_cu.MemAddressReserve(&v.uc, v.size, 0, 0, 0) == CUDA_SUCCESS;
    if (good) good = g_cu.MemMap(v.uc, v.size, 0, v.mem, 0) == CUDA_SUCCESS;
    if (good) good = g_cu.MemSetAccess(v.uc, v.size, &ad, 1) == CUDA_SUCCESS;
    if (good) good = g_cu.MemAddressReserve(&v.mcva, v.size, 0, 0, 0) == CUDA_SUCCESS;
    if (good) good = g_cu.MemMap(v.mcva, v.size, 0, v.mc, 0) == CUDA_SUCCESS;
    if (good) good = g_cu.MemSetAccess(v.mcva, v.size, &ad, 1) == CUDA_SUCCESS;
    TRY(agree(good, &all));
  }
  if (!all) {
    nvls_release(c);
    return FW_OK;
  }
  v.active = true;
  v.world = W;
  *ok = true;
  return FW_OK;
}

template <typename T, int MODE>
int run_nccl_persistent(Ctx &c, Rounds<T, MODE> &rk, cudaStream_t st, const Events &e) {
  const int W = rk.world, self = c.rank;
  if (W > kMaxRanks) return fail(FW_EINVAL, "persistent multi-GPU solve: at most %d ranks", kMaxRanks);
  const int64_t n_pad = rk.n_pad;
  const int Tn = (int)(n_pad / 128);
  const size_t rb = ((size_t)n_pad * n_pad * sizeof(T) + 255) / 256 * 256, pb = (size_t)Tn * Tn * sizeof(int);
  int *d_bar = rk.errflags() + 4;   // d_flags[4]: a scratch int for the barrier all-reduce
  auto barrier = [&]() -> int {
    NCC(c, g_nccl.AllReduce(d_bar, d_bar, 1, ncclInt32, ncclMax, c.comm, st));
    return FW_OK;
  };
  bool mc = false;
  c.last_nvls = false;
  if (W > 1 || c.nvls_opt == 1) TRY(nvls_setup(c, rb + pb, W, self, d_bar, st, &mc));
  if (getenv("FW_DEBUG")) fprintf(stderr, "[fw] persistent over a communicator: %s publish\n", mc ? "NVLS multicast" : "IPC peer-ring");
  if (mc) {   // every ring is bound to the multicast object: no IPC exchange, one store per publish
    std::vector<RankView> v(W);
    char *uc = reinterpret_cast<char *>(c.nvls.uc), *mca = reinterpret_cast<char *>(c.nvls.mcva);
    for (int q = 0; q < W; ++q) {
      int64_t r0, nr;
      partition(n_pad, W, q, &r0, &nr);
      v[q] = RankView{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, r0, (int)(r0 / 128),
                      (int)((r0 + nr) / 128)};
    }
    v[self] = RankView{rk.D, rk.P, nullptr, reinterpret_cast<int *>(uc + rb), uc, mca,
                       reinterpret_cast<int *>(mca + rb), v[self].row0, v[self].t0, v[self].t1};
    CU(cudaMemsetAsync(uc + rb, 0, pb, st));
    c.last_nvls = true;
    return launch_persistent<T, MODE>(c, v, rk.ld, n_pad, rk.maxkey, st, e, self, barrier);
  }
  TRY(c.ws_ring.ensure(rb + pb));
  // exchange the ring allocations' IPC handles (every solve: 64 B per rank; mapped once per change)
  TRY(c.ws_ipc.ensure((size_t)W * sizeof(cudaIpcMemHandle_t) * 2));
  cudaIpcMemHandle_t h;
  CU(cudaIpcGetMemHandle(&h, c.ws_ring.p));
  char *dh = static_cast<char *>(c.ws_ipc.p);
  CU(cudaMemcpyAsync(dh, &h, sizeof h, cudaMemcpyHostToDevice, st));
  NCC(c, g_nccl.AllGather(dh, dh + W * sizeof h, sizeof h, ncclChar, c.comm, st));
  std::vector<cudaIpcMemHandle_t> all(W);
  CU(cudaMemcpyAsync(all.data(), dh + W * sizeof h, W * sizeof h, cudaMemcpyDeviceToHost, st));
  TRY(sync_stream(c, st));
  if ((int)c.peer_ring.size() != W) {
    c.peer_ring.assign(W, nullptr);
    c.peer_handle.assign(W, cudaIpcMemHandle_t{});
  }
  for (int q = 0; q < W; ++q) {
    if (q == self) continue;
    if (c.peer_ring[q] && memcmp(&c.peer_handle[q], &all[q], sizeof h) == 0) continue;
    if (c.peer_ring[q]) cudaIpcCloseMemHandle(c.peer_ring[q]);
    c.peer_ring[q] = nullptr;
    CU(cudaIpcOpenMemHandle(&c.peer_ring[q], all[q], cudaIpcMemLazyEnablePeerAccess));
    c.peer_handle[q] = all[q];
  }
  std::vector<RankView> v(W);
  for (int q = 0; q < W; ++q) {
    int64_t r0, nr;
    partition(n_pad, W, q, &r0, &nr);
    char *ring = q == self ? static_cast<char *>(c.ws_ring.p) : static_cast<char *>(c.peer_ring[q]);
    v[q] = RankView{nullptr, nullptr, nullptr, reinterpret_cast<int *>(ring + rb), ring, nullptr, nullptr, r0,
                    (int)(r0 / 128), (int)((r0 + nr) / 128)};
  }
  v[self].D = rk.D;
  v[self].P = rk.P;
  CU(cudaMemsetAsync(static_cast<char *>(c.ws_ring.p) + rb, 0, pb, st));
  return launch_persistent<T, MODE>(c, v, rk.ld, n_pad, rk.maxkey, st, e, self, barrier);
}

// Loopback partition (every rank of a W-way block-row partition in this process, one GPU) as ONE
// persistent grid with the fused publish: each rank's own rows, its own ring (the pivot-row
// history the owners publish into) and pub flags. Tests the multi-GPU publish / poll protocol.
template <typename T, int MODE>
int run_loopback_persistent(Ctx &c, std::vector<Rounds<T, MODE>> &rk, cudaStream_t st, const Events &e) {
  const int W = (int)rk.size();
  const int64_t n_pad = rk[0].n_pad;
  const size_t rb = (size_t)n_pad * n_pad * sizeof(T);
  TRY(c.ws_ring.ensure(rb * W));
  std::vector<RankView> v(W);
  for (int r = 0; r < W; ++r) {
    void *ring = static_cast<char *>(c.ws_ring.p) + rb * r;
    v[r] = RankView{rk[r].D, rk[r].P, nullptr, nullptr, ring, nullptr, nullptr, rk[r].row0,
                    (int)(rk[r].row0 / 128), (int)((rk[r].row0 + rk[r].nrows) / 128)};
  }
  return launch_persistent<T, MODE>(c, v, rk[0].ld, n_pad, maxkey_of(rk), st, e);
}

template <typename T, int MODE>
int run_rounds(Ctx &c, std::vector<Part<T>> &parts, Transport tr, int world, int64_t n, int BS,
               int R, int *maxkey, int *done, cudaStream_t st, const Events &ev, bool la) {
  const int64_t n_pad = (n + 127) / 128 * 128;
  std::vector<Rounds<T, MODE>> rk;
  for (auto &p : parts) {
    rk.push_back(Rounds<T, MODE>{c, world, p.D, p.P, p.ld, n, n_pad, p.row0, p.nrows, BS, R, maxkey,
                                 {p.strip[0], p.strip[1]}, done + (tr == T_LOOPBACK ? rk.size() * R : 0)});
  }
  c.last_pairs = false;
  c.last_pdl = false;
  c.last_persist = false;
  c.last_nvls = false;
  if (tr == T_LOOPBACK && c.persistent == 1 && BS == 128 && (int)rk.size() <= kMaxRanks) {
    c.last_persist = true;
    return run_loopback_persistent<T, MODE>(c, rk, st, ev);
  }
  if (tr == T_NCCL && c.persistent == 1 && BS == 128 && world <= kMaxRanks) {
    c.last_persist = true;
    return run_nccl_persistent<T, MODE>(c, rk[0], st, ev);
  }
  if (tr != T_LOCAL) {   // the multi-rank driver: pairs when every pair of blocks sits on one rank
    const bool pairs = MODE != MODE_TAG && c.pairs && la && BS == 128 && R % 2 == 0 && R >= 4 &&
                       pairs_aligned(n, world);
    c.last_pairs = pairs;
    return run_team<T, MODE>(c, rk, tr == T_NCCL, st, ev, la, pairs);
  }
  if (use_persistent(c, MODE, tr, BS, n_pad, rk[0].row0, rk[0].nrows)) {
    c.last_persist = true;
    return run_persistent<T, MODE>(c, rk[0].D, rk[0].P, rk[0].ld, n_pad, maxkey, st, ev);
  }
  if (MODE != MODE_TAG && c.pairs && la && tr == T_LOCAL && BS == 128 && R % 2 == 0 && R >= 4 &&
      rk[0].row0 == 0 && rk[0].nrows == n_pad) {
    c.last_pairs = true;
    return rk[0].run_pairs(st, ev);
  }
  return rk[0].run(st, ev, la);
}

template <typename T, int MODE, typename S>
int run_init(cudaStream_t st, const S *src, int64_t ld_src, int64_t nsrc, int64_t n, int64_t row0,
             T *D, int32_t *P, int64_t ld, int64_t nrows, int64_t n_pad) {
  if (nrows == 0) return FW_OK;
  dim3 g((unsigned)std::min<int64_t>((n_pad / 4 + 255) / 256, 64), (unsigned)std::min<int64_t>(nrows, 2048));
  init_kernel<T, MODE, S><<<g, 256, 0, st>>>(src, ld_src, nsrc, n, row0, D, P, ld, n_pad, nrows);
  ++g_launches;
  CU(cudaGetLastError());
  return FW_OK;
}

template <typename T>
constexpr bool is_int_v() { return std::is_integral<T>::value; }

// One entry of a solve's plan: P method, compute type, whether the key range is guaranteed,
// and the largest stored key (bit pattern) a speculative key run may leave.
struct Attempt {
  int mode;
  bool f32;          // relax in FP32 (INT32 data whose stored values are integers < 2^24)
  bool key_static;
  int key_limit;
};

int key_limit_f32() {
  const float f = (float)(kKeyMaxF32 * kKeyMul + kKeyMask);
  int b;
  memcpy(&b, &f, 4);
  return b;
}

// Domain checks on the validation flags ([0] flags, [1] max weight bits) and the solve's plan:
// exact arg-min keys for integer-valued data within the key range (static, or speculative and
// verified by the max stored key), else round tags; INT32 data runs in FP32 when every value
// it can store is an integer below 2^24 (keys: max key checked).
int make_plan(bool int_t, bool want_p, const int *h_flags, int64_t n, std::vector<Attempt> *out) {
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
  const bool integral = int_t || !(h_flags[0] & 2);
  const bool has_inf = (h_flags[0] & 4) != 0;
  const double path_max = (double)(n > 1 ? n - 1 : 1) * maxw;   // bound on any finite distance
  const bool f32_exact = int_t && path_max < 16777216.0;         // 2^24: PLAIN / TAG in FP32
  std::vector<Attempt> &plan = *out;
  plan.clear();
  if (want_p && integral) {
    if (int_t && maxw <= (double)kKeyMaxF32)
      plan.push_back({MODE_KEY, true, !has_inf || path_max <= (double)kKeyMaxF32, key_limit_f32()});
    const int64_t kmax = int_t ? kKeyMaxI32 : kKeyMaxF32;
    if (maxw <= (double)kmax && !(int_t && plan.size() && plan[0].key_static))
      plan.push_back({MODE_KEY, false, !has_inf || path_max <= (double)kmax,
                      int_t ? (int)(kKeyMaxI32 * kKeyMul + kKeyMask) : key_limit_f32()});
  }
  if (want_p && (plan.empty() || !plan.back().key_static)) plan.push_back({MODE_TAG, f32_exact, true, 0});
  if (!want_p) plan.push_back({MODE_PLAIN, f32_exact, true, 0});
  return FW_OK;
}

// The parts' working buffers viewed in compute type C (same 4-byte slots).
template <typename C, typename T>
std::vector<Part<C>> view_as(const std::vector<Part<T>> &parts) {
  static_assert(sizeof(C) == sizeof(T), "same element size");
  std::vector<Part<C>> v;
  for (const auto &p : parts) {
    Part<C> q{};
    q.src = reinterpret_cast<C *>(p.src);
    q.ld_src = p.ld_src;
    q.next = p.next;
    q.ld_next = p.ld_next;
    q.rank = p.rank;
    q.row0 = p.row0;
    q.nrows = p.nrows;
    q.nsrc = p.nsrc;
    q.D = reinterpret_cast<C *>(p.D);
    q.P = p.P;
    q.ld = p.ld;
    q.inplace = p.inplace;
    q.strip[0] = reinterpret_cast<C *>(p.strip[0]);
    q.strip[1] = reinterpret_cast<C *>(p.strip[1]);
    v.push_back(q);
  }
  return v;
}

// Init (pad, diagonal, key encoding; source type T converted to compute type C) and the
// R rounds of one attempt. from_backup: re-read W from the backup of an in-place solve.
template <typename C, typename T>
int run_attempt(Ctx &c, std::vector<Part<T>> &parts, std::vector<Part<C>> &cv, Transport tr, int world,
                int64_t n, int BS, int R, int mode, bool from_backup, int *maxkey, int *done,
                cudaStream_t st, const Events &ev, bool la, cudaEvent_t e_init) {
  const int64_t n_pad = (n + 127) / 128 * 128;
  for (size_t i = 0; i < parts.size(); ++i) {
    const Part<T> &p = parts[i];
    Part<C> &q = cv[i];
    const T *isrc = (from_backup && p.backup) ? p.backup : p.src;
    const int64_t ild = (from_backup && p.backup) ? n : p.ld_src;
    switch (mode) {
      case MODE_PLAIN: TRY((run_init<C, MODE_PLAIN, T>(st, isrc, ild, p.nsrc, n, p.row0, q.D, q.P, q.ld, q.nrows, n_pad))); break;
      case MODE_TAG: TRY((run_init<C, MODE_TAG, T>(st, isrc, ild, p.nsrc, n, p.row0, q.D, q.P, q.ld, q.nrows, n_pad))); break;
      default: TRY((run_init<C, MODE_KEY, T>(st, isrc, ild, p.nsrc, n, p.row0, q.D, q.P, q.ld, q.nrows, n_pad)));
    }
  }
  CU(cudaMemsetAsync(done, 0, 4 * (size_t)R * cv.size(), st));
  CU(cudaEventRecord(e_init, st));
  switch (mode) {
    case MODE_PLAIN: return run_rounds<C, MODE_PLAIN>(c, cv, tr, world, n, BS, R, maxkey, done, st, ev, la);
    case MODE_TAG: return run_rounds<C, MODE_TAG>(c, cv, tr, world, n, BS, R, maxkey, done, st, ev, la);
    default: return run_rounds<C, MODE_KEY>(c, cv, tr, world, n, BS, R, maxkey, done, st, ev, la);
  }
}

// Epilogue passes (reading R9/R10): keys -> distances; round tags -> last k (gathering and
// transposing the final D); last k -> next hop and the sentinels.
template <typename T>
int post_pass(Ctx &c, std::vector<Part<T>> &parts, Transport tr, int world, int64_t n, int BS, int mode,
              int path_mode, int *d_flags, cudaStream_t st, bool transposed = false) {
  const int64_t n_pad = (n + 127) / 128 * 128;
  const bool nccl = tr == T_NCCL;
  // keyed mode: keys -> distances inside finalize_paths_kernel (decode = 1); keys only exist
  // with P (want_p), so the finalize pass always runs then
  if (mode == MODE_TAG && path_mode >= 0) {
    // the search reads column segments D[kb..kb+BS)[j] of rows wherever they live: the final D
    // transposed into block panels (transpose_panels_kernel: each segment one contiguous
    // 4*BS-byte read). Multi-GPU: each rank transposes ONLY its own rows — their panels are one
    // contiguous range of Dt — and the ranks exchange panel ranges with grouped broadcasts, so
    // no rank gathers the row-major D or transposes more than its rows.
    TRY(c.ws_tr.ensure((size_t)n_pad * n_pad * sizeof(T)));
    T *Dt = static_cast<T *>(c.ws_tr.p);
    auto transpose = [&](const T *src, int64_t ld, int64_t rows, int64_t g0) -> int {
      if (rows == 0) return FW_OK;
      dim3 g((unsigned)(n_pad / 32), (unsigned)(rows / 32));
      auto kern = BS == 32 ? transpose_panels_kernel<T, 32>
                           : BS == 64 ? transpose_panels_kernel<T, 64> : transpose_panels_kernel<T, 128>;
      kern<<<g, dim3(32, 8), 0, st>>>(src, ld, rows, n_pad, g0, Dt);
      CU(cudaGetLastError());
      ++g_launches;
      return FW_OK;
    };
    if (transposed) {
      // host pipeline: the caller transposed the final D once for all chunks
    } else if (nccl) {
      Part<T> &p = parts[0];
      TRY(transpose(p.D, p.ld, p.nrows, p.row0));
      NCC(c, g_nccl.GroupStart());
      for (int r = 0; r < world; ++r) {
        int64_t r0, nr;
        partition(n, world, r, &r0, &nr);
        if (nr == 0) continue;
        T *dst = Dt + r0 * n_pad;   // the panels of rows [r0, r0 + nr)
        NCC(c, g_nccl.Broadcast(dst, dst, (size_t)nr * n_pad, is_int_v<T>() ? ncclInt32 : ncclFloat32, r,
                                c.comm, st));
        ++g_bcasts;
        g_bcast_bytes += (double)nr * (double)n_pad * sizeof(T);
      }
      NCC(c, g_nccl.GroupEnd());
    } else {   // one GPU, or every rank of the loopback: the rows are one n_pad x n_pad matrix
      TRY(transpose(parts[0].D - (tr == T_LOOPBACK ? parts[0].row0 * n_pad : 0), parts[0].ld, n_pad, 0));
    }
    const size_t rb = (size_t)n_pad * sizeof(T);
    const int use_smem = rb <= 200 * 1024;
    {                        // four lanes per element
      auto launchq = [&](auto kern) -> int {
        TRY(smem_attr((const void *)kern, 200 * 1024));
        for (auto &p : parts) {
          if (p.nsrc == 0) continue;
          kern<<<(unsigned)p.nsrc, 512, use_smem ? rb : 0, st>>>(p.D, Dt, p.ld, n_pad, p.row0, n, n_pad, p.P);
          CU(cudaGetLastError());
          ++g_launches;
        }
        return FW_OK;
      };
      switch (BS * 2 + use_smem) {
        case 64: TRY(launchq(resolve_lastk_quad_kernel<T, 32, false>)); break;
        case 65: TRY(launchq(resolve_lastk_quad_kernel<T, 32, true>)); break;
        case 128: TRY(launchq(resolve_lastk_quad_kernel<T, 64, false>)); break;
        case 129: TRY(launchq(resolve_lastk_quad_kernel<T, 64, true>)); break;
        case 256: TRY(launchq(resolve_lastk_quad_kernel<T, 128, false>)); break;
        default: TRY(launchq(resolve_lastk_quad_kernel<T, 128, true>));
      }
    }
  }
  if (path_mode >= 0) {
    const size_t row_bytes = (size_t)n * sizeof(int32_t);
    const int use_smem = row_bytes <= 200 * 1024;
    TRY(smem_attr((const void *)finalize_paths_kernel<T>, 200 * 1024));
    for (auto &p : parts) {
      if (p.nsrc == 0) continue;
      finalize_paths_kernel<T><<<(unsigned)p.nsrc, 1024, use_smem ? row_bytes : 0, st>>>(
          p.D, p.P, p.ld, p.row0, n, path_mode == 0, use_smem, d_flags, is_key(mode) ? 1 : 0);
      ++g_launches;
      CU(cudaGetLastError());
    }
  }
  return FW_OK;
}

template <typename T>
int place_parts(Ctx &c, std::vector<Part<T>> &parts, Transport tr, int64_t n, int BS, bool want_p,
                bool may_retry, cudaStream_t st);
template <typename T>
int solve_placed(Ctx &c, std::vector<Part<T>> &parts, Transport tr, int world, int64_t n, int BS,
                 cudaStream_t st, const std::vector<Attempt> &plan, int *d_flags, int *h_flags,
                 int64_t bcasts0, double bcast_bytes0);

// Solve over `parts` (one part = one rank's rows): T_LOCAL (one GPU, all rows), T_NCCL (this
// process's rank of an NCCL communicator), T_LOOPBACK (every rank emulated here).
template <typename T>
int solve_parts(Ctx &c, std::vector<Part<T>> &parts, Transport tr, int world, int64_t n, int BS,
                cudaStream_t st) {
  const bool int_t = is_int_v<T>();
  const bool want_p = parts[0].next != nullptr;
  const bool nccl = tr == T_NCCL;
  Nvtx nv_solve("fw_solve");
  const int64_t bcasts0 = g_bcasts;
  const double bcast_bytes0 = g_bcast_bytes;

  // 1. validation (read-only; outputs untouched on error), reduced over all ranks
  const int R = (int)((n + BS - 1) / BS);  // rounds wholly inside the padding are skipped
  TRY(c.scratch.ensure(64 + 4 * (size_t)R * parts.size()));
  // [0] flags [1] max weight [2] max key [3] placement status; [16..16+R*W) look-ahead counters
  // (R per emulated rank of the loopback transport, W = parts.size(); R otherwise)
  int *d_flags = static_cast<int *>(c.scratch.p);
  CU(cudaMemsetAsync(d_flags, 0, 16, st));
  c.pending = false;
  if (c.async && tr == T_LOCAL && !c.in_host_entry) {
    // asynchronous device solve: no validation and no host round trip — the caller guarantees
    // the domain (fw.h). The round-tag plan is valid for every such input: FP32 data relax in
    // FP32 (bitwise the keyed result for integer data: every sum of integers < 2^24 is exact),
    // INT32 data in INT32; P through round tags and the post-pass.
    std::vector<Attempt> plan{{want_p ? MODE_TAG : MODE_PLAIN, !int_t, true, 0}};
    int h_flags[4] = {0, 0, 0, 0};
    TRY(place_parts(c, parts, tr, n, BS, want_p, false, st));
    return solve_placed<T>(c, parts, tr, world, n, BS, st, plan, d_flags, h_flags, bcasts0, bcast_bytes0);
  }
  for (auto &p : parts) {
    if (p.nsrc == 0) continue;
    const dim3 g((unsigned)std::max<int64_t>(1, std::min<int64_t>((n / 4 + 255) / 256, 16)),
                 (unsigned)std::min<int64_t>(p.nsrc, 148 * 8));
    validate_kernel<T><<<g, 256, 0, st>>>(p.src, p.ld_src, p.nsrc, n, p.row0, d_flags, d_flags + 1);
    ++g_launches;
    CU(cudaGetLastError());
  }
  // flag bits are combined with max: the rank holding a bit holds the max value as well
  if (nccl) NCC(c, g_nccl.AllReduce(d_flags, d_flags, 2, ncclInt32, ncclMax, c.comm, st));
  int h_flags[4] = {0, 0, 0, 0};
  CU(cudaMemcpyAsync(h_flags, d_flags, sizeof h_flags, cudaMemcpyDeviceToHost, st));
  TRY(sync_stream(c, st));
  std::vector<Attempt> plan;
  TRY(make_plan(int_t, want_p, h_flags, n, &plan));

  // 3. placement; over a communicator every rank learns whether all ranks placed their
  //    workspaces before the first broadcast (a rank that failed to allocate must not leave its
  //    peers waiting in a collective)
  int place_rc = place_parts(c, parts, tr, n, BS, want_p, plan.size() > 1, st);
  if (nccl) {
    std::string place_err = g_err;
    CU(cudaMemsetAsync(d_flags + 3, place_rc != FW_OK ? 1 : 0, 1, st));
    NCC(c, g_nccl.AllReduce(d_flags + 3, d_flags + 3, 1, ncclInt32, ncclMax, c.comm, st));
    CU(cudaMemcpyAsync(h_flags, d_flags, sizeof h_flags, cudaMemcpyDeviceToHost, st));
    TRY(sync_stream(c, st));
    if (place_rc != FW_OK) return fail(place_rc, "%s", place_err.c_str());
    if (h_flags[3]) return fail(FW_ENOMEM, "another rank failed to place its workspaces");
  }
  TRY(place_rc);
  return solve_placed<T>(c, parts, tr, world, n, BS, st, plan, d_flags, h_flags, bcasts0, bcast_bytes0);
}

// Workspaces of the parts: the loopback workspace, or this rank's rows in place / padded, the
// strip receive buffers of a communicator rank, and the backup of W for a speculative key run.
template <typename T>
int place_parts(Ctx &c, std::vector<Part<T>> &parts, Transport tr, int64_t n, int BS, bool want_p,
                bool may_retry, cudaStream_t st) {
  const int64_t n_pad = (n + 127) / 128 * 128;
  const bool nccl = tr == T_NCCL;
  if (tr == T_LOOPBACK) {
    // one padded n_pad x n_pad workspace: each part uses its own rows of it
    TRY(c.ws_d.ensure((size_t)n_pad * n_pad * sizeof(T)));
    if (want_p) TRY(c.ws_t.ensure((size_t)n_pad * n_pad * sizeof(int32_t)));
    const size_t sb = (size_t)(BS == 128 ? 2 : 1) * BS * n_pad * sizeof(T);   // pairs: rows a, b
    TRY(c.ws_s.ensure(2 * sb * parts.size()));
    for (size_t r = 0; r < parts.size(); ++r) {
      Part<T> &p = parts[r];
      p.ld = n_pad;
      p.D = static_cast<T *>(c.ws_d.p) + p.row0 * n_pad;
      p.P = want_p ? static_cast<int32_t *>(c.ws_t.p) + p.row0 * n_pad : nullptr;
      p.strip[0] = reinterpret_cast<T *>(static_cast<char *>(c.ws_s.p) + 2 * r * sb);
      p.strip[1] = reinterpret_cast<T *>(static_cast<char *>(c.ws_s.p) + (2 * r + 1) * sb);
    }
  } else {
    Part<T> &p = parts[0];
    p.inplace = p.nsrc == p.nrows && n == n_pad && p.ld_src == n && ((uintptr_t)p.src % 16 == 0) &&
                (!want_p || (p.ld_next == n && (uintptr_t)p.next % 16 == 0));
    p.D = p.src;
    p.P = p.next;
    p.ld = n;
    if (!p.inplace) {
      TRY(c.ws_d.ensure((size_t)std::max<int64_t>(p.nrows, 1) * n_pad * sizeof(T)));
      p.D = static_cast<T *>(c.ws_d.p);
      if (want_p) {
        TRY(c.ws_t.ensure((size_t)std::max<int64_t>(p.nrows, 1) * n_pad * sizeof(int32_t)));
        p.P = static_cast<int32_t *>(c.ws_t.p);
      }
      p.ld = n_pad;
    }
    if (!want_p) p.P = nullptr;
    if (nccl) {
      const size_t sb = (size_t)(BS == 128 ? 2 : 1) * BS * n_pad * sizeof(T);   // pairs: rows a, b
      TRY(c.ws_s.ensure(2 * sb));
      p.strip[0] = static_cast<T *>(c.ws_s.p);
      p.strip[1] = reinterpret_cast<T *>(static_cast<char *>(c.ws_s.p) + sb);
    }
    // a speculative key run may have to be redone: keep W when solving in place
    if (may_retry && p.inplace && p.nsrc > 0) {
      TRY(c.ws_b.ensure((size_t)p.nsrc * n * sizeof(T)));
      p.backup = static_cast<T *>(c.ws_b.p);
      CU(cudaMemcpy2DAsync(p.backup, n * sizeof(T), p.src, p.ld_src * sizeof(T), n * sizeof(T),
                           p.nsrc, cudaMemcpyDeviceToDevice, st));
    }
  }
  return FW_OK;
}

// The solve after validation and placement: the plan's attempts, the post-pass, unpad, stats.
template <typename T>
int solve_placed(Ctx &c, std::vector<Part<T>> &parts, Transport tr, int world, int64_t n, int BS,
                 cudaStream_t st, const std::vector<Attempt> &plan, int *d_flags, int *h_flags,
                 int64_t bcasts0, double bcast_bytes0) {
  const bool int_t = is_int_v<T>();
  const int64_t n_pad = (n + 127) / 128 * 128;
  const bool want_p = parts[0].next != nullptr;
  const bool lastk = (c.flags & FW_PATH_LAST_K) != 0;
  const int path_mode = want_p ? (lastk ? 1 : 0) : -1;
  const bool timing = (c.flags & FW_TIMING) != 0 && tr != T_LOOPBACK;
  const bool nccl = tr == T_NCCL;
  const int R = (int)((n + BS - 1) / BS);
  int *d_done = d_flags + 16;
  TRY(ensure_events(c, 4 + 3 * (size_t)R + 2 * (size_t)R));
  cudaEvent_t e_begin = c.events[0], e_end = c.events[1], e_init = c.events[2],
              e_post = c.events[3];
  Events ev{timing, c.events.data() + 4, c.events.data() + 4 + 3 * (size_t)R};
  int *d_maxkey = d_flags + 2;
  const bool la = c.lookahead && BS == 128 && R >= 2;

  // 4. attempts: the first that is exact wins (plan built above); FP32 compute for INT32 data
  //    whose stored values stay below 2^24
  const int64_t launches0 = g_launches - (int64_t)parts.size();   // + the validation launches
  CU(cudaEventRecord(e_begin, st));
  CU(cudaStreamWaitEvent(c.side, e_begin, 0));   // the side stream follows the caller's stream
  std::vector<Part<float>> fview = view_as<float>(parts);
  Attempt used = plan[0];
  for (size_t a = 0; a < plan.size(); ++a) {
    used = plan[a];
    const bool from_backup = a > 0;
    if (used.f32)
      TRY((run_attempt<float, T>(c, parts, fview, tr, world, n, BS, R, used.mode, from_backup, d_maxkey,
                                 d_done, st, ev, la, e_init)));
    else
      TRY((run_attempt<T, T>(c, parts, parts, tr, world, n, BS, R, used.mode, from_backup, d_maxkey,
                             d_done, st, ev, la, e_init)));
    if (!is_key(used.mode) || used.key_static) break;
    if (nccl) NCC(c, g_nccl.AllReduce(d_maxkey, d_maxkey, 1, ncclInt32, ncclMax, c.comm, st));
    CU(cudaMemcpyAsync(h_flags, d_flags, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
    TRY(sync_stream(c, st));
    if (getenv("FW_DEBUG"))
      fprintf(stderr, "fwb: speculative key run: max stored key bits %d, limit %d\n", h_flags[2], used.key_limit);
    if (h_flags[2] <= used.key_limit || a + 1 == plan.size()) break;
    CU(cudaMemsetAsync(d_maxkey, 0, 4, st));   // a stored key left the exact range: next plan
  }
  const int mode = used.mode;

  // 5. epilogue passes in the compute type; FP32 results of INT32 data back to INT32
  if (used.f32) {
    TRY(post_pass<float>(c, fview, tr, world, n, BS, mode, path_mode, d_flags, st));
    if (!std::is_same<T, float>::value)
      for (auto &p : fview) {
        if (p.nsrc == 0) continue;
        dim3 g((unsigned)std::min<int64_t>((n + 255) / 256, 64), (unsigned)std::min<int64_t>(p.nsrc, 65535));
        f32_to_i32_kernel<<<g, 256, 0, st>>>(p.D, p.ld, n, p.nsrc);
        ++g_launches;
        CU(cudaGetLastError());
      }
  } else {
    TRY(post_pass<T>(c, parts, tr, world, n, BS, mode, path_mode, d_flags, st));
  }
  CU(cudaEventRecord(e_post, st));

  // 6. unpad into the caller's buffers
  for (auto &p : parts) {
    if (p.inplace || p.nsrc == 0) continue;
    dim3 g((unsigned)std::min<int64_t>((n + 255) / 256, 64), (unsigned)std::min<int64_t>(p.nsrc, 65535));
    unpad_kernel<T><<<g, 256, 0, st>>>(p.D, p.ld, n, p.src, p.ld_src, p.nsrc);
    ++g_launches;
    CU(cudaGetLastError());
    if (want_p) {
      unpad_kernel<int32_t><<<g, 256, 0, st>>>(p.P, p.ld, n, p.next, p.ld_next, p.nsrc);
      ++g_launches;
      CU(cudaGetLastError());
    }
  }
  CU(cudaEventRecord(e_end, st));
  if (c.async && tr == T_LOCAL && !c.in_host_entry) {   // everything is enqueued: return without waiting
    fw_stats s{};
    s.n = n;
    s.n_pad = n_pad;
    s.block = BS;
    s.rounds = R;
    s.is_int = int_t;
    s.path_mode = path_mode;
    s.p_method = used.mode;
    s.compute_f32 = (used.f32 || !int_t) ? 1 : 0;
    s.persistent = c.last_persist ? (c.last_nvls ? 2 : 1) : 0;
    s.kernel_launches = g_launches - launches0;
    c.stats = s;
    c.has_stats = true;
    c.pending = true;
    c.pending_st = st;
    return FW_OK;
  }
  CU(cudaMemcpyAsync(h_flags, d_flags, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
  TRY(sync_stream(c, st));
  if (h_flags[0] & 16)
    return fail(FW_ECUDA, "a look-ahead wait timed out (wait_count_kernel): the results are not valid");
  if (h_flags[0] & 32)
    return fail(FW_ECUDA, "a persistent-kernel dependency wait timed out: the results are not valid");
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
  s.compute_f32 = (used.f32 || !int_t) ? 1 : 0;
  float ms = 0.f;
  CU(cudaEventElapsedTime(&ms, e_begin, e_end));
  s.solve_ms = ms;
  // bulk phase-3 launches issued: one per pair of rounds with pairs, else one per round
  s.phase3_launches = c.last_persist ? 1 : c.last_pairs ? R / 2 : R;
  s.persistent = c.last_persist ? (c.last_nvls ? 2 : 1) : 0;
  s.broadcasts = g_bcasts - bcasts0;
  s.bcast_bytes = g_bcast_bytes - bcast_bytes0;
  s.kernel_launches = g_launches - launches0;
  // phase-3 relaxations of this process's rows: rows and columns outside the round's strips
  double relax = 0;
  for (auto &p : parts)
    for (int K = 0; K < R; ++K) {
      const int64_t kb = (int64_t)K * BS;
      const double rows = (double)p.nrows - ((kb >= p.row0 && kb < p.row0 + p.nrows) ? BS : 0);
      relax += rows * (double)(n_pad - BS) * BS;
    }
  if (c.last_pairs) {  // every pair relaxes all local tiles outside its strip region through 256 k
    relax = 0;
    for (auto &p : parts)
      for (int Pp = 0; Pp < R / 2; ++Pp) {
        const int64_t kb = (int64_t)Pp * 2 * BS;
        const double rows = (double)p.nrows - ((kb >= p.row0 && kb < p.row0 + p.nrows) ? 2 * BS : 0);
        relax += rows * (double)(n_pad - 2 * BS) * (2.0 * BS);
      }
  }
  if (c.last_persist)  // one launch does every phase: n_pad^3 relaxations (phases 1, 2 and 3)
    relax = (double)n_pad * (double)n_pad * (double)n_pad;
  s.phase3_relaxations = relax;
  if (timing && c.last_persist) {
    auto at = [&](cudaEvent_t e) {
      float t = 0.f;
      cudaEventElapsedTime(&t, e_begin, e);
      return (double)t;
    };
    s.phase3_ms = at(ev.ev[2]) - at(ev.ev[0]);   // the persistent launch (all phases)
    s.phase1_ms = at(ev.ev[0]) - at(e_init);
    s.post_ms = at(e_post) - at(ev.ev[2]);
  } else if (timing && !c.last_pairs && c.last_pdl) {   // phase-3 launches overlap: timed as one span
    auto at = [&](cudaEvent_t e) {
      float t = 0.f;
      cudaEventElapsedTime(&t, e_begin, e);
      return (double)t;
    };
    for (int K = 0; K < R; ++K) {
      const double p1 = at(ev.ev[3 * K]), p2 = at(ev.ev[3 * K + 1]);
      s.phase1_ms += p1 - (K > 0 ? at(ev.sync[2 * K]) : at(e_init));
      s.phase2_ms += p2 - p1;
    }
    const double p3e = at(ev.ev[3 * (R - 1) + 2]);
    s.phase3_ms = p3e - at(ev.ev[1]);
    s.post_ms = at(e_post) - p3e;
  } else if (timing && c.last_pairs && c.last_pdl) {   // bulk launches overlap: timed as one span
    auto at = [&](cudaEvent_t e) {
      float t = 0.f;
      cudaEventElapsedTime(&t, e_begin, e);
      return (double)t;
    };
    const int NP = R / 2;
    const double p3s = at(ev.ev[0]), p3e = at(ev.ev[3 * (NP - 1) + 2]);
    s.phase1_ms = p3s - at(e_init);   // the first pair's pivot path
    s.phase3_ms = p3e - p3s;
    for (int Pp = 0; Pp + 1 < NP; ++Pp) s.phase2_ms += at(ev.sync[2 * Pp + 1]) - at(ev.sync[2 * Pp]);
    s.post_ms = at(e_post) - p3e;
  } else if (timing && c.last_pairs) {
    auto at = [&](cudaEvent_t e) {
      float t = 0.f;
      cudaEventElapsedTime(&t, e_begin, e);
      return (double)t;
    };
    double prev = at(e_init);
    for (int Pp = 0; Pp < R / 2; ++Pp) {
      const double p3s = at(ev.ev[3 * Pp]), p3e = at(ev.ev[3 * Pp + 2]);
      s.phase3_ms += p3e - p3s;
      s.phase1_ms += p3s - prev;     // pivot path not hidden under the previous pair (phases 1-2 + strip3)
      if (Pp + 1 < R / 2) s.phase2_ms += at(ev.sync[2 * Pp + 1]) - at(ev.sync[2 * Pp]);   // pivot path of the next pair, side stream
      prev = p3e;
    }
    s.post_ms = at(e_post) - prev;
  } else if (timing) {
    // absolute event times (ms since e_begin); with the look-ahead, phases 1-2 of round K
    // run on the side stream from the wait for round K-1's look-ahead tiles, concurrently
    // with the rest of round K-1's phase 3
    auto at = [&](cudaEvent_t e) {
      float t = 0.f;
      cudaEventElapsedTime(&t, e_begin, e);
      return (double)t;
    };
    double prev_p3_end = at(e_init);
    for (int K = 0; K < R; ++K) {
      const double p1 = at(ev.ev[3 * K]), p2 = at(ev.ev[3 * K + 1]), p3 = at(ev.ev[3 * K + 2]);
      const double p1_start = (la && K > 0) ? at(ev.sync[2 * K]) : prev_p3_end;
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

// This process's rows as one part (T_LOCAL: all rows; T_NCCL: the communicator rank's rows).
template <typename T>
int solve_rows(Ctx &c, T *src, int64_t ld_src, int32_t *next, int64_t ld_next, int64_t n, int BS,
               cudaStream_t st) {
  const int world = c.comm ? c.world : 1;
  const int rank = c.comm ? c.rank : 0;
  Part<T> p{};
  p.src = src; p.ld_src = ld_src; p.next = next; p.ld_next = ld_next; p.rank = rank;
  partition(n, world, rank, &p.row0, &p.nrows);
  p.nsrc = std::max<int64_t>(0, std::min(p.nrows, n - p.row0));
  std::vector<Part<T>> parts{p};
  // a communicator of any size (one rank included) takes the NCCL data plane
  return solve_parts<T>(c, parts, c.comm ? T_NCCL : T_LOCAL, world, n, BS, st);
}

// Every rank of a `world`-way partition emulated in this process (loopback transport).
template <typename T>
int solve_loopback(Ctx &c, T *src, int64_t ld_src, int32_t *next, int64_t ld_next, int64_t n,
                   int BS, int world, cudaStream_t st) {
  std::vector<Part<T>> parts;
  for (int r = 0; r < world; ++r) {
    Part<T> p{};
    p.rank = r;
    partition(n, world, r, &p.row0, &p.nrows);
    p.nsrc = std::max<int64_t>(0, std::min(p.nrows, n - p.row0));
    p.src = src + std::min(p.row0, n) * ld_src;
    p.ld_src = ld_src;
    p.next = next ? next + std::min(p.row0, n) * ld_next : nullptr;
    p.ld_next = ld_next;
    parts.push_back(p);
  }
  return solve_parts<T>(c, parts, T_LOOPBACK, world, n, BS, st);
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

// ---- host <-> device copies --------------------------------------------------------------------
// Pinned host buffers go straight to the copy engine. Pageable ones go through a ring of pinned
// staging slices; the host side of each slice (pageable <-> pinned) is copied by a small pool
// of threads (one memcpy thread reaches ~11 GB/s here, PCIe ~53 GB/s).
class CopyPool {
 public:
  static CopyPool &get() {
    static CopyPool pool;
    return pool;
  }
  void copy(void *dst, const void *src, size_t bytes) {
    // one parallel copy at a time (rank threads of a team solve share the pool): when the pool
    // is busy, or the copy is small, the calling thread copies alone
    std::unique_lock<std::mutex> busy(call_mu_, std::try_to_lock);
    if (bytes < (4u << 20) || nth_ == 0 || !busy.owns_lock()) {
      memcpy(dst, src, bytes);
      return;
    }
    std::unique_lock<std::mutex> lk(mu_);
    dst_ = static_cast<char *>(dst);
    src_ = static_cast<const char *>(src);
    bytes_ = bytes;
    const size_t parts = (size_t)nth_ + 1;
    part_ = ((bytes + parts - 1) / parts + 63) & ~size_t(63);   // parts * part_ >= bytes
    pending_ = nth_;
    ++gen_;
    cv_.notify_all();
    lk.unlock();
    run_part(0);                                  // the caller copies part 0
    lk.lock();
    done_.wait(lk, [&] { return pending_ == 0; });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto &t : th_) t.join();
  }

 private:
  CopyPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const char *e = getenv("FW_COPY_THREADS");   // tuning: helper threads of the host copy pool
    nth_ = e ? std::max(0, atoi(e)) : (int)std::min(15u, hw > 2 ? hw * 3 / 4 - 1 : 0u);   // 11 of 16 cores
    for (int w = 1; w <= nth_; ++w) th_.emplace_back([this, w] { loop(w); });
  }
  void run_part(int w) {
    const size_t lo = std::min(bytes_, (size_t)w * part_), hi = std::min(bytes_, lo + part_);
    if (hi > lo) memcpy(dst_ + lo, src_ + lo, hi - lo);
  }
  void loop(int w) {
    int seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      if (stop_) return;
      lk.unlock();
      run_part(w);
      lk.lock();
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> th_;
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_;
  char *dst_ = nullptr;
  const char *src_ = nullptr;
  size_t bytes_ = 0, part_ = 0;
  int nth_ = 0, gen_ = 0, pending_ = 0;
  bool stop_ = false;
};

constexpr int kSlots = 4;                       // staging ring: kSlots slices of kSlice bytes
constexpr size_t kSlice = 32ull << 20;

int ring_slot(Ctx &c, char **slot, int *idx) {
  TRY(ensure_pinned(c, kSlots * kSlice));
  while (c.ring_ev.size() < (size_t)kSlots) {
    cudaEvent_t e;
    CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c.ring_ev.push_back(e);
    c.ring_used.push_back(false);
  }
  const int s = c.ring_pos++ % kSlots;
  if (c.ring_used[s]) CU(cudaEventSynchronize(c.ring_ev[s]));   // its last copy is done
  *slot = static_cast<char *>(c.pinned) + (size_t)s * kSlice;
  *idx = s;
  return FW_OK;
}

// Enqueue an H2D copy on st. Pageable sources are staged slice by slice (the host returns once
// the last slice is in the ring; the ring's events keep the slices alive until copied).
int host_h2d(Ctx &c, void *dst, const void *src, size_t bytes, cudaStream_t st, bool pinned) {
  if (pinned) {
    CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    return FW_OK;
  }
  for (size_t off = 0; off < bytes; off += kSlice) {
    const size_t len = std::min(kSlice, bytes - off);
    char *slot = nullptr;
    int s = 0;
    TRY(ring_slot(c, &slot, &s));
    CopyPool::get().copy(slot, static_cast<const char *>(src) + off, len);
    CU(cudaMemcpyAsync(static_cast<char *>(dst) + off, slot, len, cudaMemcpyHostToDevice, st));
    CU(cudaEventRecord(c.ring_ev[s], st));
    c.ring_used[s] = true;
  }
  return FW_OK;
}

// D2H of `rows` rows of `width` bytes (device pitch spitch -> host pitch dpitch) on st. Pinned:
// enqueued only. Pageable: staged, and the data is in dst when this returns (the DMA of the next
// slice overlaps the host copy of the previous one).
int host_d2h(Ctx &c, void *dst, size_t dpitch, const void *src, size_t spitch, size_t width, size_t rows,
             cudaStream_t st, bool pinned) {
  if (rows == 0 || width == 0) return FW_OK;
  if (!pinned && width > kSlice) return fail(FW_EINVAL, "host_d2h: row of %zu bytes > staging slice", width);
  if (pinned) {
    CU(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, cudaMemcpyDeviceToHost, st));
    return FW_OK;
  }
  const size_t per = std::max<size_t>(1, kSlice / width);
  int prev = -1;
  size_t prev_r = 0, prev_n = 0;
  char *prev_slot = nullptr;
  auto drain = [&]() -> int {
    if (prev < 0) return FW_OK;
    CU(cudaEventSynchronize(c.ring_ev[prev]));
    for (size_t r = 0; r < prev_n; ++r) {        // contiguous rows: one parallel copy
      if (dpitch == width) {
        CopyPool::get().copy(static_cast<char *>(dst) + prev_r * dpitch, prev_slot, prev_n * width);
        break;
      }
      memcpy(static_cast<char *>(dst) + (prev_r + r) * dpitch, prev_slot + r * width, width);
    }
    prev = -1;
    return FW_OK;
  };
  for (size_t r0 = 0; r0 < rows; r0 += per) {
    const size_t nr = std::min(per, rows - r0);
    char *slot = nullptr;
    int s = 0;
    TRY(ring_slot(c, &slot, &s));
    CU(cudaMemcpy2DAsync(slot, width, static_cast<const char *>(src) + r0 * spitch, spitch, width, nr,
                         cudaMemcpyDeviceToHost, st));
    CU(cudaEventRecord(c.ring_ev[s], st));
    c.ring_used[s] = true;
    TRY(drain());
    prev = s;
    prev_r = r0;
    prev_n = nr;
    prev_slot = slot;
  }
  return drain();
}

int copy_h2d(Ctx &c, void *dst, const void *src, size_t bytes, cudaStream_t st) {
  TRY(host_h2d(c, dst, src, bytes, st, is_pinned(src)));
  CU(cudaStreamSynchronize(st));
  return FW_OK;
}

int copy_d2h(Ctx &c, void *dst, const void *src, size_t bytes, cudaStream_t st) {
  // as rows of kSlice bytes (+ a tail row): host_d2h stages whole rows per slice
  const bool pinned = is_pinned(dst);
  const size_t rows = bytes / kSlice, tail = bytes - rows * kSlice;
  TRY(host_d2h(c, dst, kSlice, src, kSlice, kSlice, rows, st, pinned));
  TRY(host_d2h(c, static_cast<char *>(dst) + rows * kSlice, tail, static_cast<const char *>(src) + rows * kSlice,
               tail, tail, tail ? 1 : 0, st, pinned));
  CU(cudaStreamSynchronize(st));
  return FW_OK;
}

// ---- host pipeline: copies overlapped with the solve (one GPU, pinned host buffers) ----------
// DESIGN.md §4.8, reading R16. The rows are split into chunks (tile-row boundaries
// t_0 = 0 < t_1 < .. < t_C); chunk c holds the pivots of rounds [t_c, t_c+1) (BS = 128).
//   arrival    c = 0..C-1: H2D + validation of chunk c on the copy stream; init and rounds
//              [0, t_c+1) of chunk c, in order, on the compute stream. The pivots of rounds
//              < t_c belong to earlier chunks, which completed those rounds on arrival; chunk c
//              computes its own pivots. Each row runs its rounds in order and reads pivot
//              strips that have completed the round: values are lengths of real paths and only
//              decrease, so "after round K, D[i][j] <= the shortest i->j path through blocks
//              <= K" holds as in the standard schedule.
//   check      every chunk validated: the plan taken from chunk 0's flags must be the plan of
//              the whole matrix, else the pipelined work is dropped and the standard solve runs
//              (nothing has been written to the caller's buffers yet).
//   departure  c = C-1..0: chunk c is final (its arrival did rounds < t_c+1, the steps before
//              did every later block on it): emit its D out of place, run its P post-pass,
//              D2H on the copy stream; meanwhile the rows [0, t_c) (one launch per round)
//              run the rounds of block range [t_c, t_c+1), whose pivots (chunk c) are FINAL.
//              With final pivots the remaining blocks may come in any order: on a shortest
//              i->j path, let v be the first intermediate in a block not yet done; after the
//              arrival D[i][v] <= |i..v| (all its intermediates lie in done blocks), and the
//              round of v's block sets D[i][j] <= D[i][v] + D[v][j] = |i..j|. Keys / last k
//              stay valid (D[i][j] = D[i][k] + D[k][j] on the final D, the triangle argument).
// The last chunk departs as soon as the arrival ends; chunk 0 (small) departs last, so only
// its copy is exposed. Chunk sizes grow geometrically so the arrival has work as soon as the
// first chunk lands and most launches cover many tile-rows.
struct PipeGeom {
  int64_t n, n_pad, ld;
  int BS, R;
  std::vector<int> tb;   // chunk boundaries in tile-rows: tb[0] = 0 .. tb[C] = n_pad / 128
  bool pinned_d = true, pinned_p = true;   // host buffers pinned (else staged through the ring)
  int nchunks() const { return (int)tb.size() - 1; }
  int64_t rows_of(int t) const { return (int64_t)t * 128; }
  int kend(int c) const { return (int)std::min<int64_t>(R, tb[c + 1]); }   // rounds [0, kend) on arrival
  int64_t nsrc(int c) const {
    return std::max<int64_t>(0, std::min<int64_t>(rows_of(tb[c + 1]), n) - rows_of(tb[c]));
  }
};

int pipe_events(Ctx &c, size_t count) {
  while (c.pev.size() < count) {
    cudaEvent_t e;
    CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c.pev.push_back(e);
  }
  return FW_OK;
}

// H2D + validation of chunk ci on the copy stream; pev[ci] = landed. A pageable source is
// staged through the pinned ring (the host returns once the chunk is in flight).
template <typename T>
int pipe_arrive(Ctx &c, const PipeGeom &g, int ci, const T *dist_h, T *raw, int *d_flags) {
  const int64_t r0 = g.rows_of(g.tb[ci]), nsrc = g.nsrc(ci);
  if (nsrc > 0) {
    TRY(host_h2d(c, raw + r0 * g.n, dist_h + r0 * g.n, (size_t)nsrc * g.n * sizeof(T), c.copy, g.pinned_d));
    const dim3 gr((unsigned)std::max<int64_t>(1, std::min<int64_t>((g.n / 4 + 255) / 256, 16)),
                  (unsigned)std::min<int64_t>(nsrc, 148 * 8));
    validate_kernel<T><<<gr, 256, 0, c.copy>>>(raw + r0 * g.n, g.n, nsrc, g.n, r0, d_flags, d_flags + 1);
    ++g_launches;
    CU(cudaGetLastError());
  }
  CU(cudaEventRecord(c.pev[ci], c.copy));
  return FW_OK;
}

// Everything after chunk 0's flags chose the plan `spec` (compute type C, P mode MODE).
template <typename C, int MODE, typename T>
int pipe_solve(Ctx &c, const PipeGeom &g, T *dist_h, int32_t *next_h, T *raw, C *D, int32_t *P,
               int *d_flags, int *h_flags, const Attempt &spec, int path_mode, bool *fallback,
               cudaEvent_t e_comp_end) {
  const int NC = g.nchunks();
  cudaStream_t st = c.stream;
  int *d_done = d_flags + 16;
  const Events ev{false, c.events.data() + 4, c.events.data() + 4 + 3 * (size_t)g.R};
  const bool la = c.lookahead && g.BS == 128;
  // rounds [K0, K1) on tile-rows [t0, t1), pivot strips read in place from the whole matrix:
  // rounds whose pivots lie outside the rows as plain phase-3 launches + one column-strip batch,
  // the rows' own rounds with their pivot phases and the look-ahead
  bool even_bounds = true;
  for (int t : g.tb) even_bounds = even_bounds && t % 2 == 0;
  auto run = [&](int t0, int t1, int K0, int K1) -> int {
    if (t1 <= t0 || K1 <= K0) return FW_OK;
    const int64_t r0 = g.rows_of(t0);
    Rounds<C, MODE> rk{c, 1, D + r0 * g.ld, P ? P + r0 * g.ld : nullptr, g.ld, g.n, g.n_pad, r0,
                       g.rows_of(t1 - t0), g.BS, g.R, d_flags + 2, {nullptr, nullptr}, d_done, D};
    const int own0 = std::max(K0, std::min(K1, t0)), own1 = std::max(own0, std::min(K1, t1));
    // a fused pair (K, K+1) needs both pivot blocks complete through K+1: they must lie in one
    // chunk, which holds when every chunk boundary is even
    const bool plain_pairs = c.pairs && t1 - t0 >= c.pipe_pair_rows && even_bounds;
    TRY(rk.run_plain(st, K0, own0, plain_pairs));    // pivots in earlier rows
    if (own1 > own0) {                               // own pivots: pairs of rounds (§4.9) or one by one
      // (pairs only on wide row ranges: below 32 tile-rows the two sub-rounds of pivot phases
      // take longer than the bulk launch they hide under)
      if (MODE != MODE_TAG && c.pairs && la && own0 % 2 == 0 && (own1 - own0) % 2 == 0 && t1 - t0 >= c.pipe_pair_rows) {
        TRY(rk.run_pairs(st, ev, own0, own1));
      } else {
        CU(cudaMemsetAsync(d_done, 0, 4 * (size_t)g.R, st));
        TRY(rk.run(st, ev, la, own0, own1));
      }
    }
    return rk.run_plain(st, own1, K1, plain_pairs);  // pivots in later rows
  };
  // arrival: init + rounds [0, t_c+1) of each chunk as it lands; the next chunk is put in flight
  // after this one's work is queued (a pageable copy keeps the host busy meanwhile)
  for (int ci = 0; ci < NC; ++ci) {
    const int64_t r0 = g.rows_of(g.tb[ci]);
    CU(cudaStreamWaitEvent(st, c.pev[ci], 0));
    TRY((run_init<C, MODE, T>(st, raw + r0 * g.n, g.n, g.nsrc(ci), g.n, r0, D + r0 * g.ld,
                              P ? P + r0 * g.ld : nullptr, g.ld, g.rows_of(g.tb[ci + 1] - g.tb[ci]),
                              g.n_pad)));
    TRY(run(g.tb[ci], g.tb[ci + 1], 0, g.kend(ci)));
    if (ci + 1 < NC) TRY(pipe_arrive<T>(c, g, ci + 1, dist_h, raw, d_flags));
  }
  // check: the whole matrix's plan must be the speculated one
  CU(cudaMemcpyAsync(h_flags, d_flags, 4 * sizeof(int), cudaMemcpyDeviceToHost, c.copy));
  CU(cudaStreamSynchronize(c.copy));
  std::vector<Attempt> plan;
  const int rc = make_plan(std::is_integral<T>::value, next_h != nullptr, h_flags, g.n, &plan);
  if (rc != FW_OK || plan[0].mode != spec.mode || plan[0].f32 != spec.f32 ||
      plan[0].key_static != spec.key_static) {
    CU(cudaStreamSynchronize(st));
    CU(cudaStreamSynchronize(c.side));
    if (rc == FW_OK) *fallback = true;
    return rc;
  }
  // departure, (a) all compute: for c = C-1..0 chunk c is final -> its P post-pass, D emitted out
  // of place (event pev[NC + c], max-key snapshot), then rows [0, t_c) take block range c.
  // A speculative key run (keys not statically exact) is checked before each chunk leaves: the
  // chunk's values came from sums of keys stored so far, exact iff the running max key is in
  // range then (it only grows). Its D is emitted into a separate buffer so the input survives
  // for the standard solve if a check fails.
  const bool check_keys = is_key(MODE) && !spec.key_static;
  T *out = check_keys ? static_cast<T *>(c.ws_b.p) : raw;
  TRY(smem_attr((const void *)finalize_paths_kernel<C>, 200 * 1024));
  for (int ci = NC - 1; ci >= 0; --ci) {
    const int64_t r0 = g.rows_of(g.tb[ci]), nsrc = g.nsrc(ci);
    if (nsrc > 0) {
      if (path_mode >= 0 && MODE != MODE_TAG) {   // TAG: P needs the whole final D (after the loop)
        const size_t row_bytes = (size_t)g.n * sizeof(int32_t);
        const int use_smem = row_bytes <= 200 * 1024;
        finalize_paths_kernel<C><<<(unsigned)nsrc, 1024, use_smem ? row_bytes : 0, st>>>(
            D + r0 * g.ld, P + r0 * g.ld, g.ld, r0, g.n, path_mode == 0, use_smem, d_flags, 0);
        ++g_launches;
        CU(cudaGetLastError());
      }
      const dim3 gr((unsigned)std::min<int64_t>((g.n + 255) / 256, 64), (unsigned)std::min<int64_t>(nsrc, 65535));
      emit_rows_kernel<C, T><<<gr, 256, 0, st>>>(D + r0 * g.ld, g.ld, g.n, nsrc, out + r0 * g.n, g.n,
                                                 is_key(MODE) ? 1 : 0);
      ++g_launches;
      CU(cudaGetLastError());
      if (check_keys)
        CU(cudaMemcpyAsync(c.pin_small + ci, d_flags + 2, sizeof(int), cudaMemcpyDeviceToHost, st));
      CU(cudaEventRecord(c.pev[NC + ci], st));
    }
    TRY(run(0, g.tb[ci], g.tb[ci], g.kend(ci)));
  }
  // round tags -> last k (reading R9: valid for any round order, the last improvement in time
  // wrote the tag) -> next hop, on the whole final D (transposed once), per row chunk of
  // kTagRows rows so each chunk's P copy overlaps the next chunk's search
  constexpr int64_t kTagRows = 2048;
  const bool tag_p = MODE == MODE_TAG && path_mode >= 0;
  const int ntag = tag_p ? (int)((g.n + kTagRows - 1) / kTagRows) : 0;
  for (int q = 0; q < ntag; ++q) {
    const int64_t r0 = q * kTagRows;
    std::vector<Part<C>> part(1);
    part[0].D = D + r0 * g.ld;
    part[0].P = P + r0 * g.ld;
    part[0].ld = g.ld;
    part[0].row0 = r0;
    part[0].nrows = std::min<int64_t>(kTagRows, g.n_pad - r0);
    part[0].nsrc = std::min<int64_t>(kTagRows, g.n - r0);
    if (q == 0) {   // the transpose of the whole final D (the search reads column segments)
      TRY(c.ws_tr.ensure((size_t)g.n_pad * g.n_pad * sizeof(C)));
      dim3 gt((unsigned)(g.n_pad / 32), (unsigned)(g.n_pad / 32));
      transpose_panels_kernel<C, 128><<<gt, dim3(32, 8), 0, st>>>(D, g.ld, g.n_pad, g.n_pad, 0,
                                                                static_cast<C *>(c.ws_tr.p));   // pipeline: BS = 128
      CU(cudaGetLastError());
      ++g_launches;
    }
    TRY(post_pass<C>(c, part, T_LOCAL, 1, g.n, g.BS, MODE_TAG, path_mode, d_flags, st, true));
    CU(cudaEventRecord(c.pev[2 * NC + q], st));
  }
  CU(cudaEventRecord(e_comp_end, st));
  // departure, (b) the copies out, in the same order: the host waits for a chunk only where it
  // must (a key check, or a pageable destination staged through the ring)
  for (int ci = NC - 1; ci >= 0; --ci) {
    const int64_t r0 = g.rows_of(g.tb[ci]), nsrc = g.nsrc(ci);
    if (nsrc == 0) continue;
    if (check_keys) {
      CU(cudaEventSynchronize(c.pev[NC + ci]));
      if (c.pin_small[ci] > spec.key_limit) {   // a stored key left the exact range
        CU(cudaStreamSynchronize(st));
        CU(cudaStreamSynchronize(c.side));
        CU(cudaStreamSynchronize(c.copy));
        *fallback = true;
        return FW_OK;
      }
    }
    CU(cudaStreamWaitEvent(c.copy, c.pev[NC + ci], 0));
    const size_t rb = (size_t)g.n * sizeof(T);
    TRY(host_d2h(c, dist_h + r0 * g.n, rb, out + r0 * g.n, rb, rb, nsrc, c.copy, g.pinned_d));
    if (path_mode >= 0 && MODE != MODE_TAG)
      TRY(host_d2h(c, next_h + r0 * g.n, g.n * sizeof(int32_t), P + r0 * g.ld, g.ld * sizeof(int32_t),
                   g.n * sizeof(int32_t), nsrc, c.copy, g.pinned_p));
  }
  for (int q = 0; q < ntag; ++q) {
    const int64_t r0 = q * kTagRows, nsrc = std::min<int64_t>(kTagRows, g.n - r0);
    CU(cudaStreamWaitEvent(c.copy, c.pev[2 * NC + q], 0));
    TRY(host_d2h(c, next_h + r0 * g.n, g.n * sizeof(int32_t), P + r0 * g.ld, g.ld * sizeof(int32_t),
                 g.n * sizeof(int32_t), nsrc, c.copy, g.pinned_p));
  }
  CU(cudaStreamWaitEvent(c.copy, e_comp_end, 0));
  return FW_OK;
}

template <typename C, typename T>
int pipe_dispatch(Ctx &c, const PipeGeom &g, T *dist_h, int32_t *next_h, T *raw, int *d_flags,
                  int *h_flags, const Attempt &spec, int path_mode, bool *fallback, cudaEvent_t e_comp_end) {
  C *D = static_cast<C *>(c.ws_d.p);
  int32_t *P = path_mode >= 0 ? static_cast<int32_t *>(c.ws_t.p) : nullptr;
  if (spec.mode == MODE_KEY)
    return pipe_solve<C, MODE_KEY, T>(c, g, dist_h, next_h, raw, D, P, d_flags, h_flags, spec, path_mode,
                                      fallback, e_comp_end);
  if (spec.mode == MODE_TAG)
    return pipe_solve<C, MODE_TAG, T>(c, g, dist_h, next_h, raw, D, P, d_flags, h_flags, spec, path_mode,
                                      fallback, e_comp_end);
  return pipe_solve<C, MODE_PLAIN, T>(c, g, dist_h, next_h, raw, D, nullptr, d_flags, h_flags, spec,
                                      path_mode, fallback, e_comp_end);
}

// Chunk boundaries (tile-rows) of the host pipeline; empty = no pipeline. Auto (pipe_tiles < 0):
// at n >= 8192, chunks of 8, 8, 16, 32, .. tile-rows (doubling; the last takes the rest); at
// 4096 <= n < 8192 two halves (C2: 11.4 -> 10.4 ms per fw_solve); below, none.
// pipe_tiles = k > 0: uniform chunks of k tile-rows when there are at least two.
std::vector<int> pipe_bounds_of(int64_t n, int pipe_tiles, int pipe_first) {
  const int tiles = (int)((n + 127) / 128);
  std::vector<int> tb;
  if (pipe_tiles == 0) return tb;
  if (pipe_tiles > 0) {
    if (tiles < 2 * pipe_tiles) return tb;
    for (int t = 0; t < tiles; t += pipe_tiles) tb.push_back(t);
    tb.push_back(tiles);
    return tb;
  }
  if (tiles >= 32 && tiles < 64) return {0, tiles / 2, tiles};   // small n: two halves
  if (tiles < 64 || pipe_first < 1 || 2 * pipe_first > tiles) return tb;
  tb.push_back(0);
  int t = pipe_first, step = pipe_first;
  tb.push_back(t);
  while (t + 2 * step < tiles) {   // the next chunk would not be the last: keep doubling
    t += step;
    tb.push_back(t);
    step *= 2;
  }
  tb.push_back(tiles);
  return tb;
}
std::vector<int> pipe_bounds(const Ctx &c, int64_t n) { return pipe_bounds_of(n, c.pipe_tiles, c.pipe_first); }

// Pipelined host solve; returns FW_OK with *done = false when the standard path must run, and
// *raw_ready = true when the caller's input is then already on the device (c.user_d, n x n).
template <typename T>
int solve_host_pipelined(Ctx &c, T *dist, int32_t *next, int64_t n, int BS, bool *done, bool *raw_ready) {
  *done = false;
  *raw_ready = false;
  PipeGeom g{};
  g.tb = pipe_bounds(c, n);
  if (g.tb.size() < 3 || BS != 128) return FW_OK;
  g.pinned_d = is_pinned(dist);
  g.pinned_p = next ? is_pinned(next) : true;
  g.n = n;
  g.n_pad = (n + 127) / 128 * 128;
  g.ld = g.n_pad;
  g.BS = BS;
  g.R = (int)((n + BS - 1) / BS);
  const int path_mode = next ? ((c.flags & FW_PATH_LAST_K) ? 1 : 0) : -1;
  const bool want_p = next != nullptr;
  if (!c.copy) CU(cudaStreamCreateWithFlags(&c.copy, cudaStreamNonBlocking));
  TRY(c.user_d.ensure((size_t)n * n * sizeof(T)));
  TRY(c.ws_d.ensure((size_t)g.n_pad * g.n_pad * sizeof(T)));
  if (want_p) TRY(c.ws_t.ensure((size_t)g.n_pad * g.n_pad * sizeof(int32_t)));
  TRY(c.scratch.ensure(64 + 4 * (size_t)g.R));
  TRY(ensure_events(c, 4 + 3 * (size_t)g.R + 2 * (size_t)g.R));
  TRY(pipe_events(c, 2 * (size_t)g.nchunks() + 40));   // + one per 2048-row tag chunk (n <= 65536)
  T *raw = static_cast<T *>(c.user_d.p);
  int *d_flags = static_cast<int *>(c.scratch.p);
  cudaEvent_t e_begin = c.events[0], e_end = c.events[1], e_land0 = c.events[2], e_comp = c.events[3];
  const int64_t launches0 = g_launches;

  // chunk 0: lands, is validated, and its flags choose the plan (speculation, checked later)
  CU(cudaEventRecord(e_begin, c.copy));
  CU(cudaMemsetAsync(d_flags, 0, 16, c.copy));
  TRY(pipe_arrive<T>(c, g, 0, dist, raw, d_flags));
  CU(cudaEventRecord(e_land0, c.copy));
  int h_flags[4] = {0, 0, 0, 0};
  CU(cudaMemcpyAsync(h_flags, d_flags, sizeof h_flags, cudaMemcpyDeviceToHost, c.copy));
  CU(cudaStreamSynchronize(c.copy));
  std::vector<Attempt> plan;
  TRY(make_plan(std::is_integral<T>::value, want_p, h_flags, n, &plan));
  const Attempt spec = plan[0];
  if (!spec.key_static) {   // speculative keys: checked per departing chunk (pipe_solve)
    TRY(c.ws_b.ensure((size_t)n * n * sizeof(T)));
    if (!c.pin_small) {
      void *p = nullptr;
      if (cudaHostAlloc(&p, 64 * 1024, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        return fail(FW_ENOMEM, "cudaHostAlloc(64 KiB) failed");
      }
      c.pin_small = static_cast<int *>(p);
    }
    if (g.nchunks() > 16 * 1024) return FW_OK;
  }
  CU(cudaStreamWaitEvent(c.stream, e_begin, 0));
  CU(cudaStreamWaitEvent(c.side, e_begin, 0));

  bool fallback = false;
  int rc = spec.f32 ? pipe_dispatch<float, T>(c, g, dist, next, raw, d_flags, h_flags, spec, path_mode,
                                              &fallback, e_comp)
                    : pipe_dispatch<T, T>(c, g, dist, next, raw, d_flags, h_flags, spec, path_mode,
                                          &fallback, e_comp);
  if (rc != FW_OK) return rc;
  if (fallback) {   // every chunk landed and user_d still holds the input
    *raw_ready = true;
    return FW_OK;
  }
  CU(cudaEventRecord(e_end, c.copy));
  CU(cudaStreamSynchronize(c.copy));
  CU(cudaMemcpy(h_flags, d_flags, sizeof h_flags, cudaMemcpyDeviceToHost));
  if (h_flags[0] & 16)
    return fail(FW_ECUDA, "a look-ahead wait timed out (wait_count_kernel): the results are not valid");
  if (h_flags[0] & 8)
    return fail(FW_ERANGE, "next-hop resolution did not converge (zero-weight cycle?)");

  fw_stats s{};
  s.n = n;
  s.n_pad = g.n_pad;
  s.block = BS;
  s.rounds = g.R;
  s.is_int = std::is_integral<T>::value;
  s.path_mode = path_mode;
  s.p_method = spec.mode;
  s.compute_f32 = (spec.f32 || !std::is_integral<T>::value) ? 1 : 0;
  float ms = 0.f;
  CU(cudaEventElapsedTime(&ms, e_begin, e_end));
  s.solve_ms = ms;
  CU(cudaEventElapsedTime(&ms, e_begin, e_land0));
  s.h2d_ms = ms;                        // exposed: until chunk 0 has landed
  CU(cudaEventElapsedTime(&ms, e_comp, e_end));
  s.d2h_ms = ms;                        // exposed: after the last chunk's compute
  s.phase3_relaxations = (double)g.R * (double)(g.n_pad - BS) * (double)(g.n_pad - BS) * BS;
  s.kernel_launches = g_launches - launches0;
  s.host_chunks = g.nchunks();
  c.stats = s;
  c.has_stats = true;
  *done = true;
  return FW_OK;
}

// ---- single-process multi-GPU (fw_solve with ngpus > 1) ---------------------------------
// One context per device (its own streams, workspaces, staging), an NCCL communicator over the
// devices (ncclCommInitAll), and one host thread per device running the same per-rank driver
// as the one-process-per-GPU path (solve_rows over the communicator rank's block-rows).
int ctx_setup(Ctx *c, int dev, unsigned flags, bool lookahead) {
  CU(cudaSetDevice(dev));
  c->dev = dev;
  c->flags = flags;
  c->lookahead = lookahead;
  CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  int prio_lo = 0, prio_hi = 0;
  CU(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  CU(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, prio_hi));
  return FW_OK;
}

void ctx_release(Ctx *c) {
  cudaSetDevice(c->dev);
  cudaDeviceSynchronize();
  for (Ctx *t : c->team) {
    ctx_release(t);
    delete t;
  }
  c->team.clear();
  cudaSetDevice(c->dev);
  if (c->comm) g_nccl.CommDestroy(c->comm);
  c->comm = nullptr;
  nvls_release(*c);
  for (void *pr : c->peer_ring)
    if (pr) cudaIpcCloseMemHandle(pr);
  c->peer_ring.clear();
  c->peer_handle.clear();
  for (DevBuf *b : {&c->ws_d, &c->ws_t, &c->ws_b, &c->ws_s, &c->ws_tr, &c->user_d,
                    &c->user_t, &c->scratch, &c->ws_ver, &c->ws_ring, &c->ws_ipc})
    b->release();
  if (c->pinned) cudaFreeHost(c->pinned);
  c->pinned = nullptr;
  c->pinned_bytes = 0;
  if (c->pin_small) cudaFreeHost(c->pin_small);
  c->pin_small = nullptr;
  for (auto e : c->events) cudaEventDestroy(e);
  c->events.clear();
  for (auto e : c->pev) cudaEventDestroy(e);
  c->pev.clear();
  for (auto e : c->ring_ev) cudaEventDestroy(e);
  c->ring_ev.clear();
  for (auto e : c->xev) cudaEventDestroy(e);
  c->xev.clear();
  for (auto e : c->lb_ev) cudaEventDestroy(e);
  c->lb_ev.clear();
  for (auto q : c->lb_st) cudaStreamDestroy(q);
  c->lb_st.clear();
  c->ring_used.clear();
  if (c->copy) cudaStreamDestroy(c->copy);
  c->copy = nullptr;
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->side) cudaStreamDestroy(c->side);
  c->stream = c->side = nullptr;
}

void team_release(Ctx &c);

int team_setup(Ctx &c, int G) {
  if ((int)c.team.size() == G) return FW_OK;
  team_release(c);
  TRY(load_nccl());
  std::vector<int> devs(G);
  for (int d = 0; d < G; ++d) {
    devs[d] = d;
    Ctx *t = new Ctx();
    c.team.push_back(t);
    TRY(ctx_setup(t, d, c.flags, c.lookahead));
    t->rank = d;
    t->world = G;
  }
  // non-blocking communicators (bounded waits, abort on failure: see nccl_settle), one per
  // device, created in one group
  ncclUniqueId uid;
  NC(g_nccl.GetUniqueId(&uid));
  std::vector<ncclComm_t> comms(G, nullptr);
  NC(g_nccl.GroupStart());
  for (int d = 0; d < G; ++d) {
    CU(cudaSetDevice(devs[d]));
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 0;
    const ncclResult_t r = g_nccl.CommInitRankConfig(&comms[d], G, uid, d, &cfg);
    if (r != ncclSuccess && r != ncclInProgress) {
      g_nccl.GroupEnd();
      return fail(FW_ENCCL, "ncclCommInitRankConfig(device %d): %s", d, g_nccl.GetErrorString(r));
    }
  }
  const ncclResult_t ge = g_nccl.GroupEnd();
  if (ge != ncclSuccess && ge != ncclInProgress)
    return fail(FW_ENCCL, "ncclGroupEnd (team init): %s", g_nccl.GetErrorString(ge));
  for (int d = 0; d < G; ++d) c.team[d]->comm = comms[d];
  for (int d = 0; d < G; ++d) TRY(nccl_settle(*c.team[d], "team communicator init"));
  CU(cudaSetDevice(c.dev));
  return FW_OK;
}

void team_release(Ctx &c) {
  for (Ctx *t : c.team) {
    ctx_release(t);
    delete t;
  }
  c.team.clear();
}

// One rank of a team solve: copy its block-rows of the host matrix in, solve, copy them out.
template <typename T>
int team_rank_solve(Ctx &t, T *dist, int32_t *next, int64_t n, int BS) {
  CU(cudaSetDevice(t.dev));
  int64_t row0, nrows;
  partition(n, t.world, t.rank, &row0, &nrows);
  const int64_t nsrc = std::max<int64_t>(0, std::min(nrows, n - row0));
  const size_t bytes = (size_t)nsrc * n * sizeof(T), pbytes = (size_t)nsrc * n * sizeof(int32_t);
  TRY(t.user_d.ensure(std::max<size_t>(bytes, 16)));
  if (next) TRY(t.user_t.ensure(std::max<size_t>(pbytes, 16)));
  T *d = static_cast<T *>(t.user_d.p);
  int32_t *tp = next ? static_cast<int32_t *>(t.user_t.p) : nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  if (bytes) TRY(copy_h2d(t, d, dist + row0 * n, bytes, t.stream));
  TRY(sync_stream(t, t.stream));
  const auto t1 = std::chrono::steady_clock::now();
  TRY(solve_rows<T>(t, d, n, tp, n, n, BS, t.stream));
  const auto t2 = std::chrono::steady_clock::now();
  if (bytes) TRY(copy_d2h(t, dist + row0 * n, d, bytes, t.stream));
  if (next && pbytes) TRY(copy_d2h(t, next + row0 * n, tp, pbytes, t.stream));
  TRY(sync_stream(t, t.stream));
  const auto t3 = std::chrono::steady_clock::now();
  t.stats.h2d_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  t.stats.d2h_ms = std::chrono::duration<double, std::milli>(t3 - t2).count();
  return FW_OK;
}

template <typename T>
int solve_host_team(Ctx &c, T *dist, int32_t *next, int64_t n, int BS, int G) {
  {
    const int rc0 = team_setup(c, G);
    if (rc0 != FW_OK) {
      const std::string e = g_err;
      team_release(c);
      return fail(rc0, "%s", e.c_str());
    }
  }
  // the first rank that fails raises the flag; its peers' bounded waits (sync_stream,
  // nccl_settle) see it and abort their communicators instead of waiting in a collective
  std::atomic<int> abort_flag{0};
  for (Ctx *t : c.team) t->abort_flag = &abort_flag;
  std::vector<int> rc(G, FW_OK);
  std::vector<std::string> err(G);
  std::vector<std::thread> th;
  for (int d = 0; d < G; ++d)
    th.emplace_back([&, d] {
      rc[d] = team_rank_solve<T>(*c.team[d], dist, next, n, BS);
      if (rc[d] != FW_OK) {
        err[d] = g_err;   // g_err is thread-local
        abort_flag.store(1);
      }
    });
  for (auto &x : th) x.join();
  for (Ctx *t : c.team) t->abort_flag = nullptr;
  cudaSetDevice(c.dev);
  int first = -1;   // the rank that failed on its own (not because a peer did), else any failed rank
  for (int d = 0; d < G; ++d)
    if (rc[d] != FW_OK && (first < 0 || (rc[first] == FW_ENCCL && rc[d] != FW_ENCCL))) first = d;
  if (first >= 0) {
    const int code = rc[first];
    const std::string msg = err[first];
    const int dev = c.team[first]->dev;
    team_release(c);   // communicators aborted or in an unknown state: rebuilt on the next call
    return fail(code, "rank %d (device %d): %s", first, dev, msg.c_str());
  }
  c.stats = c.team[0]->stats;   // rank 0's solve; host copies: the slowest rank
  for (int d = 1; d < G; ++d) {
    c.stats.h2d_ms = std::max(c.stats.h2d_ms, c.team[d]->stats.h2d_ms);
    c.stats.d2h_ms = std::max(c.stats.d2h_ms, c.team[d]->stats.d2h_ms);
    c.stats.solve_ms = std::max(c.stats.solve_ms, c.team[d]->stats.solve_ms);
  }
  c.has_stats = true;
  return FW_OK;
}

template <typename T>
int solve_host(T *dist, int32_t *next, int64_t n, int block, int ngpus) {
  int BS = 0;
  TRY(check_common(n, dist, block, &BS));
  Ctx &c = *g_ctx;
  if (ngpus == 0) ngpus = c.ngpus_max;
  if (ngpus < 1 || ngpus > c.ngpus_max)
    return fail(FW_EINVAL, "ngpus = %d outside [0, %d] (fw_init's ngpus_max / visible devices)", ngpus,
                c.ngpus_max);
  if (c.comm)
    return fail(FW_ESTATE, "a multi-GPU communicator is active: use fw_dist_solve_* or fw_comm_free");
  if (ngpus > 1) return solve_host_team<T>(c, dist, next, n, BS, ngpus);
  CU(cudaSetDevice(c.dev));
  struct HostEntry {   // the asynchronous device mode never applies to the host entry points
    Ctx &c;
    explicit HostEntry(Ctx &x) : c(x) { c.in_host_entry = true; }
    ~HostEntry() { c.in_host_entry = false; }
  } host_entry(c);
  bool piped = false, raw_ready = false;
  TRY(solve_host_pipelined<T>(c, dist, next, n, BS, &piped, &raw_ready));
  if (piped) return FW_OK;
  const size_t bytes = (size_t)n * n * sizeof(T);
  TRY(c.user_d.ensure(bytes));
  if (next) TRY(c.user_t.ensure((size_t)n * n * sizeof(int32_t)));
  T *d = static_cast<T *>(c.user_d.p);
  int32_t *t = next ? static_cast<int32_t *>(c.user_t.p) : nullptr;
  cudaEvent_t h0, h1;
  CU(cudaEventCreate(&h0));
  CU(cudaEventCreate(&h1));
  CU(cudaEventRecord(h0, c.stream));
  // after a dropped pipeline the input is already on the device (and `dist` may hold rows of D)
  int rc = raw_ready ? FW_OK : copy_h2d(c, d, dist, bytes, c.stream);
  if (rc == FW_OK) rc = (cudaEventRecord(h1, c.stream) == cudaSuccess) ? FW_OK : FW_ECUDA;
  if (rc == FW_OK) rc = solve_rows<T>(c, d, n, t, n, n, BS, c.stream);
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
int solve_dev_entry(T *d_dist, int32_t *d_next, int64_t n, int64_t ld, int block, void *stream,
                    bool dist) {
  int BS = 0;
  TRY(check_common(n, d_dist, block, &BS));
  if (ld < n) return fail(FW_EINVAL, "ld (%lld) < n (%lld)", (long long)ld, (long long)n);
  Ctx &c = *g_ctx;
  if (!dist && c.comm)
    return fail(FW_ESTATE, "a multi-GPU communicator is active: use fw_dist_solve_* or fw_comm_free");
  if (dist && c.comm == nullptr)
    return fail(c.comm_dead ? FW_ENCCL : FW_ESTATE,
                c.comm_dead ? "the communicator was aborted after an NCCL failure: fw_comm_free, then fw_comm_init"
                            : "fw_dist_solve_* needs fw_comm_init first");
  return solve_rows<T>(c, d_dist, ld, d_next, ld, n, BS, static_cast<cudaStream_t>(stream));
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
  c->ngpus_max = ngpus_max == 0 ? count : ngpus_max;
  CU(cudaGetDevice(&c->dev));
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, c->dev));
  if (prop.major != 10 || prop.minor != 0) {   // arch-specific sm_100a SASS only, no portable PTX
    delete c;
    return fail(FW_ECUDA, "device %s is sm_%d%d; this library is built for sm_100a only", prop.name,
                prop.major, prop.minor);
  }
  CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  int prio_lo = 0, prio_hi = 0;
  CU(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  CU(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, prio_hi));
  const char *la = getenv("FW_LOOKAHEAD");
  c->lookahead = !(la && la[0] == '0');
  const char *pr = getenv("FW_PAIRS");
  c->pairs = !(pr && pr[0] == '0');
  const char *pd = getenv("FW_PDL");
  c->pair_pdl = !(pd && pd[0] == '0');
  const char *po = getenv("FW_PAIR_ORDER");
  c->pair_order = !(po && po[0] == '0');
  const char *pp = getenv("FW_PIPE_PAIR_ROWS");
  if (pp && atoi(pp) >= 1) c->pipe_pair_rows = atoi(pp);
  const char *pb1 = getenv("FW_P1_BLOCKED");
  if (pb1) g_p1_blocked = atoi(pb1) != 0;
  const char *ps = getenv("FW_PERSISTENT");   // one persistent launch per solve: -1 auto, 0 off, 1 on
  if (ps && atoi(ps) >= -1 && atoi(ps) <= 1) c->persistent = atoi(ps);
  const char *pf = getenv("FW_PIPE_FIRST");   // tuning: first chunk of the auto host pipeline
  if (pf && atoi(pf) >= 1 && atoi(pf) <= 64) c->pipe_first = atoi(pf);
  g_ctx = c;
  g_err.clear();
  return FW_OK;
}

int fw_set_option(const char *name, int value) {
  if (!g_ctx) return fail(FW_ESTATE, "fw_init has not been called");
  if (!name) return fail(FW_EINVAL, "name is NULL");
  Ctx &c = *g_ctx;
  const std::string k = name;
  if (k == "lookahead") c.lookahead = value != 0;
  else if (k == "pairs") c.pairs = value != 0;
  else if (k == "pdl") c.pair_pdl = value != 0;
  else if (k == "pair_order") c.pair_order = value != 0;
  else if (k == "pipe_pair_rows" && value >= 1) c.pipe_pair_rows = value;
  else if (k == "pipe_first" && value >= 1 && value <= 64) c.pipe_first = value;
  else if (k == "persistent" && value >= -1 && value <= 1) c.persistent = value;
  else if (k == "persist_gap" && value >= -1) c.persist_gap = value;
  else if (k == "persist_relaxed" && (value == 0 || value == 1)) c.persist_relaxed = value;
  else if (k == "async" && (value == 0 || value == 1)) c.async = value != 0;
  else if (k == "persist_quarters" && value >= -1 && value <= 2) c.persist_quarters = value;
  else if (k == "persist_p1_lone" && value >= -1 && value <= 1) c.persist_p1_lone = value;
  else if (k == "persist_stage_old" && (value == 0 || value == 1)) c.persist_stage_old = value;
  else if (k == "nvls" && value >= -1 && value <= 1) c.nvls_opt = value;
  else return fail(FW_EINVAL, "unknown option or value: %s = %d", name, value);
  return FW_OK;
}

int fw_free(void) {
  if (!g_ctx) return FW_OK;
  ctx_release(g_ctx);
  delete g_ctx;
  g_ctx = nullptr;
  return FW_OK;
}

int fw_solve(float *dist, int32_t *next, int64_t n, int block, int ngpus) {
  return solve_host<float>(dist, next, n, block, ngpus);
}

int fw_set_host_pipeline(int chunk_tiles) {
  if (!g_ctx) return fail(FW_ESTATE, "fw_init has not been called");
  if (chunk_tiles < -1) return fail(FW_EINVAL, "chunk_tiles must be >= -1 (got %d)", chunk_tiles);
  g_ctx->pipe_tiles = chunk_tiles;
  return FW_OK;
}

int64_t fw_path(const int32_t *P, const void *dist, int dist_is_int32, int64_t n, int64_t i, int64_t j, int mode,
                int32_t *out, int64_t max_len) {
  if (!P || n <= 0 || n > 65536 || i < 0 || i >= n || j < 0 || j >= n || max_len < 0 || (max_len > 0 && !out) ||
      (mode != FW_PATH_NEXT_HOP && mode != FW_PATH_LAST_K) || (mode == FW_PATH_LAST_K && !dist))
    return -fail(FW_EINVAL, "fw_path: bad arguments (n=%lld i=%lld j=%lld mode=%d)", (long long)n, (long long)i,
                 (long long)j, mode);
  int64_t len = 0;
  auto emit = [&](int64_t v) -> bool {   // false once the path is longer than a simple path
    if (len < max_len) out[len] = (int32_t)v;
    return ++len <= n;
  };
  if (dist) {   // reachability from D: INF (FP32 +inf, INT32 FW_INF_I32) = no path
    const int64_t e = i * n + j;
    const bool inf = dist_is_int32 ? static_cast<const int32_t *>(dist)[e] >= FW_INF_I32
                                   : !(static_cast<const float *>(dist)[e] < INFINITY);
    if (inf) return 0;
  }
  emit(i);
  if (i == j) return 1;
  if (mode == FW_PATH_NEXT_HOP) {   // i, next[i][j], next[next[i][j]][j], ..., j
    int64_t h = i;
    while (h != j) {
      const int32_t nx = P[h * n + j];
      if (nx < 0) {
        if (h == i && !dist) return 0;   // unreachable (next = -1)
        return -fail(FW_EINVAL, "fw_path: next[%lld][%lld] = %d on the way to %lld", (long long)h, (long long)j,
                     nx, (long long)j);
      }
      if (nx >= n || !emit(nx))
        return -fail(FW_EINVAL, "fw_path: next-hop chain %lld -> %lld leaves [0, n) or exceeds n - 1 hops",
                     (long long)i, (long long)j);
      h = nx;
    }
  } else {   // LAST_K: path(i,k) + path(k,j) for k = P[i][j]; -1 = direct edge
    std::vector<std::pair<int32_t, int32_t>> stack{{(int32_t)i, (int32_t)j}};
    while (!stack.empty()) {
      const auto [a, b] = stack.back();
      stack.pop_back();
      const int32_t k = P[(int64_t)a * n + b];
      if (k < 0) {
        if (!emit(b))
          return -fail(FW_EINVAL, "fw_path: LAST_K expansion of %lld -> %lld exceeds n - 1 hops", (long long)i,
                       (long long)j);
        continue;
      }
      if (k >= n || k == a || k == b || stack.size() > (size_t)n)
        return -fail(FW_EINVAL, "fw_path: LAST_K[%d][%d] = %d is not an intermediate vertex", a, b, k);
      stack.push_back({k, b});   // expanded after (a, k)
      stack.push_back({a, k});
    }
  }
  if (len > max_len && max_len > 0)
    return -fail(FW_ERANGE, "fw_path: the path has %lld vertices > max_len = %lld", (long long)len,
                 (long long)max_len);
  return len;
}

int fw_host_pipeline_bounds(int64_t n, int chunk_tiles, int first_tiles, int32_t *out, int max_out) {
  if (n <= 0 || n > 65536 || chunk_tiles < -1 || (chunk_tiles == -1 && first_tiles < 1) || max_out < 0 ||
      (max_out > 0 && !out))
    return -fail(FW_EINVAL, "bad arguments (n=%lld chunk_tiles=%d first_tiles=%d)", (long long)n, chunk_tiles,
                 first_tiles);
  const std::vector<int> tb = pipe_bounds_of(n, chunk_tiles, first_tiles);
  if ((int)tb.size() > max_out) return -fail(FW_EINVAL, "max_out = %d < %zu bounds", max_out, tb.size());
  for (size_t i = 0; i < tb.size(); ++i) out[i] = tb[i];
  return (int)tb.size();
}

int64_t fw_persist_schedule(int64_t n, int world, int rank, int gap, uint32_t *out, int64_t max_out) {
  if (n <= 0 || n > 65536 || world < 1 || world > kMaxRanks || rank < -4 || rank >= world || gap < 0 ||
      max_out < 0 || (max_out > 0 && !out) || (rank <= -2 && world != 1))
    return -fail(FW_EINVAL, "fw_persist_schedule: bad arguments (n=%lld world=%d rank=%d gap=%d)", (long long)n, world,
                 rank, gap);
  const int64_t n_pad = (n + 127) / 128 * 128;
  const int T = (int)(n_pad / 128);
  std::vector<int> t0(world), t1(world);
  for (int r = 0; r < world; ++r) {
    int64_t r0, nr;
    partition(n_pad, world, r, &r0, &nr);
    t0[r] = (int)(r0 / 128);
    t1[r] = (int)((r0 + nr) / 128);
  }
  std::vector<unsigned> items;
  if (rank <= -2) {   // the one-GPU kernel's arithmetic decode (persist_decode), run on the host;
                      // -3: with quarter items (the quarter in the rank bits), -4: critical quarters
    PersistArgs a{};
    a.T = T;
    a.gap = gap;
    a.quarters = rank == -3 ? 1 : rank == -4 ? 2 : 0;
    const int Q = a.quarters == 1 ? 4 : 1;
    const long long total = a.quarters == 2 ? persist_total_crit(T)
                                            : 1 + (long long)Q * 2 * (T - 1) +
                                                  (long long)T * ((long long)T * T + (Q - 1) * (4LL * T - 5));
    for (long long it = 0; it < total; ++it) {
      const Item w = persist_decode(a, it);
      if (w.type != IT_NONE) items.push_back(pack_item(w.type == IT_QTILE ? w.r : 0, w.type, w.K, w.I, w.J));
    }
  } else {
    persist_items(T, world, t0, t1, rank, gap, &items);
  }
  if ((int64_t)items.size() > max_out && max_out > 0)
    return -fail(FW_EINVAL, "fw_persist_schedule: %zu items > max_out = %lld", items.size(), (long long)max_out);
  if (max_out > 0) memcpy(out, items.data(), items.size() * sizeof(unsigned));
  return (int64_t)items.size();
}

int fw_solve_i32(int32_t *dist, int32_t *next, int64_t n, int block, int ngpus) {
  return solve_host<int32_t>(dist, next, n, block, ngpus);
}

int fw_solve_device_f32(float *d_dist, int32_t *d_next, int64_t n, int64_t ld, int block,
                        void *stream) {
  return solve_dev_entry<float>(d_dist, d_next, n, ld, block, stream, false);
}

int fw_solve_device_i32(int32_t *d_dist, int32_t *d_next, int64_t n, int64_t ld, int block,
                        void *stream) {
  return solve_dev_entry<int32_t>(d_dist, d_next, n, ld, block, stream, false);
}

int fw_dist_partition(int64_t n, int world, int rank, int64_t *row0, int64_t *nrows) {
  if (n <= 0 || world <= 0 || rank < 0 || rank >= world || !row0 || !nrows)
    return fail(FW_EINVAL, "bad partition arguments (n=%lld world=%d rank=%d)", (long long)n, world, rank);
  partition(n, world, rank, row0, nrows);
  // rows the caller holds: the real rows of the range
  *nrows = std::max<int64_t>(0, std::min<int64_t>(*nrows, n - *row0));
  return FW_OK;
}

int fw_dist_owner(int64_t n, int world, int64_t row) {
  if (n <= 0 || world <= 0 || row < 0 || row >= (n + 127) / 128 * 128) return -1;
  return owner_of(n, world, row);
}

int fw_comm_unique_id(unsigned char *out) {
  if (!out) return fail(FW_EINVAL, "out is NULL");
  TRY(load_nccl());
  ncclUniqueId id;
  NC(g_nccl.GetUniqueId(&id));
  memcpy(out, &id, sizeof id);
  return FW_OK;
}

int fw_comm_init(const unsigned char *id, int rank, int world) {
  if (!g_ctx) return fail(FW_ESTATE, "fw_init has not been called");
  if (!id || world <= 0 || rank < 0 || rank >= world)
    return fail(FW_EINVAL, "bad communicator arguments (rank=%d world=%d)", rank, world);
  if (g_ctx->comm) return fail(FW_ESTATE, "a communicator is already initialised");
  TRY(load_nccl());
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof uid);
  CU(cudaSetDevice(g_ctx->dev));
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  cfg.blocking = 0;   // bounded waits: a missing or failed peer ends in FW_ENCCL, not a hang
  const ncclResult_t r = g_nccl.CommInitRankConfig(&g_ctx->comm, world, uid, rank, &cfg);
  if (r != ncclSuccess && r != ncclInProgress) {
    g_ctx->comm = nullptr;
    return fail(FW_ENCCL, "ncclCommInitRankConfig: %s", g_nccl.GetErrorString(r));
  }
  g_ctx->comm_dead = false;
  TRY(nccl_settle(*g_ctx, "communicator init"));
  g_ctx->rank = rank;
  g_ctx->world = world;
  return FW_OK;
}

int fw_comm_free(void) {
  if (!g_ctx) return FW_OK;
  if (g_ctx->comm) {
    cudaDeviceSynchronize();
    g_nccl.CommDestroy(g_ctx->comm);
  }
  nvls_release(*g_ctx);
  g_ctx->comm = nullptr;
  g_ctx->comm_dead = false;
  g_ctx->rank = 0;
  g_ctx->world = 1;
  return FW_OK;
}

int fw_dist_loopback_solve_device_f32(float *d_dist, int32_t *d_next, int64_t n, int64_t ld,
                                      int block, int world, void *stream) {
  int BS = 0;
  TRY(check_common(n, d_dist, block, &BS));
  if (ld < n) return fail(FW_EINVAL, "ld (%lld) < n (%lld)", (long long)ld, (long long)n);
  if (world < 1 || world > 64) return fail(FW_EINVAL, "world must be in [1, 64] (got %d)", world);
  return solve_loopback<float>(*g_ctx, d_dist, ld, d_next, ld, n, BS, world,
                               static_cast<cudaStream_t>(stream));
}

int fw_dist_loopback_solve_device_i32(int32_t *d_dist, int32_t *d_next, int64_t n, int64_t ld,
                                      int block, int world, void *stream) {
  int BS = 0;
  TRY(check_common(n, d_dist, block, &BS));
  if (ld < n) return fail(FW_EINVAL, "ld (%lld) < n (%lld)", (long long)ld, (long long)n);
  if (world < 1 || world > 64) return fail(FW_EINVAL, "world must be in [1, 64] (got %d)", world);
  return solve_loopback<int32_t>(*g_ctx, d_dist, ld, d_next, ld, n, BS, world,
                                 static_cast<cudaStream_t>(stream));
}

int fw_dist_solve_device_f32(float *d_rows, int32_t *d_next_rows, int64_t n, int64_t ld, int block,
                             void *stream) {
  return solve_dev_entry<float>(d_rows, d_next_rows, n, ld, block, stream, true);
}

int fw_dist_solve_device_i32(int32_t *d_rows, int32_t *d_next_rows, int64_t n, int64_t ld,
                             int block, void *stream) {
  return solve_dev_entry<int32_t>(d_rows, d_next_rows, n, ld, block, stream, true);
}

const char *fw_last_error(void) { return g_err.c_str(); }

int fw_last_stats(fw_stats *out) {
  if (!g_ctx || !g_ctx->has_stats) return fail(FW_ESTATE, "no solve has completed yet");
  if (!out) return fail(FW_EINVAL, "out is NULL");
  Ctx &c = *g_ctx;
  if (c.pending) {   // an asynchronous solve: wait for it, then its time and device-side errors
    c.pending = false;
    CU(cudaEventSynchronize(c.events[1]));
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, c.events[0], c.events[1]));
    c.stats.solve_ms = ms;
    int h[4] = {0, 0, 0, 0};
    CU(cudaMemcpy(h, c.scratch.p, sizeof h, cudaMemcpyDeviceToHost));
    if (h[0] & (16 | 32)) return fail(FW_ECUDA, "a dependency wait of the last (asynchronous) solve timed out");
    if (h[0] & 8) return fail(FW_ERANGE, "next-hop resolution of the last (asynchronous) solve did not converge");
  }
  *out = c.stats;
  return FW_OK;
}

const char *fw_version(void) { return "fwb200 0.2 sm_100a"; }

}  // extern "C"

// Phase-3 explorer, TMA variant (development tool, not part of the library).
// Same tile (128 x 128, 256 threads, 8 x 8 per thread, FADD2 + FMNMX3, keyed epilogue) as the
// library's minplus_tile_kernel, but the k-chunks are staged by the Tensor Memory Accelerator:
// one thread issues cp.async.bulk.tensor for the A chunk (128 rows x 32 k, 128-B swizzle) and
// the B chunk (32 k x 128 columns) of a stage, completion is tracked by an mbarrier per stage
// (expect_tx), and the warps release a stage through a second mbarrier instead of
// __syncthreads. No per-thread cp.async addresses: compare registers, spills and
// relaxations / clock / SM with the library kernel on the same launch (n = 16384, K-depth 128).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <vector>
#include <stdlib.h>
#include "../fw_kernels.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

constexpr int NS = 3, BK = 32, TM = 128, TN = 128;
#ifndef SWZ
#define SWZ 0
#endif
// A box: BK columns, or BK + 4 (VAR & 8: rows of 144 B, the library's conflict-free padded stride;
// the 4 extra columns are loaded and ignored)
constexpr int A_W = BK + 4;
constexpr int A_BYTES = TM * A_W * 4, B_BYTES = BK * TN * 4, ST_BYTES = A_BYTES + B_BYTES;   // 18 + 16 KB

// VAR: 1 = keyed epilogue with P (as the library's KEY mode); 2 = round-2 scheme: thread 0 alone
// waits on the stage's full mbarrier, then ONE __syncthreads per chunk (as the library's cp.async
// pipeline) releases the stage and orders the reads (no empty barriers, no per-thread waits);
// 4 = 128-B swizzled A reads (else dense 128-B rows, 2-way bank conflicts on the A loads)
template <int VAR>
__global__ void __launch_bounds__(256, 2)
p3t(float *__restrict__ D, int32_t *__restrict__ P, const __grid_constant__ CUtensorMap mapA,
    const __grid_constant__ CUtensorMap mapB, int64_t ld, int kb, int *maxkey) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char *sm = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + NS * ST_BYTES);
  uint64_t *empty = full + NS;
  const int i0 = blockIdx.y * TM, j0 = blockIdx.x * TN;
  if ((i0 + TM > kb && i0 < kb + 128) || (j0 + TN > kb && j0 < kb + 128)) return;
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16, lane = tid & 31;
  constexpr int nch = 128 / BK;
  constexpr unsigned TXB = ((VAR & 8) ? A_W : BK) * TM * 4 + B_BYTES;   // bytes one stage's TMA pair lands
  if (VAR & 16) {   // warm L2 with the epilogue's tile, as the library kernel does
    for (int l = tid; l < TM * 4; l += 256)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(D + (int64_t)(i0 + l / 4) * ld + j0 + (l % 4) * 32));
  }
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < ((VAR & 2) ? NS - 1 : NS) && s < nch; ++s) {
      mbar_expect_tx(&full[s], TXB);
      tma_2d(sm + s * ST_BYTES, &mapA, kb + s * BK, i0, &full[s]);
      tma_2d(sm + s * ST_BYTES + A_BYTES, &mapB, j0, kb + s * BK, &full[s]);
    }
  }
  float acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = __int_as_float(0x7f800000);
  const int sw = ty & 7;   // 128-B swizzle: 16-B chunk q of row r sits at chunk q ^ (r & 7); r & 7 == ty & 7
#pragma unroll 1
  for (int ch = 0; ch < nch; ++ch) {
    const int s = ch % NS;
    if (VAR & 2) {
      if (tid == 0) mbar_wait(&full[s], (ch / NS) & 1);
      __syncthreads();   // chunk ch visible to all; every warp is past chunk ch-1
      if (tid == 0 && ch + NS - 1 < nch) {   // chunk ch+2 into the stage chunk ch-1 used (free at ch = 0)
        const int s2 = (ch + NS - 1) % NS;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&full[s2], TXB);
        tma_2d(sm + s2 * ST_BYTES, &mapA, kb + (ch + NS - 1) * BK, i0, &full[s2]);
        tma_2d(sm + s2 * ST_BYTES + A_BYTES, &mapB, j0, kb + (ch + NS - 1) * BK, &full[s2]);
      }
    } else {
      mbar_wait(&full[s], (ch / NS) & 1);
    }
    constexpr int ARB = (VAR & 8) ? A_W * 4 : BK * 4;                        // A row pitch (bytes)
    const unsigned char *as = sm + s * ST_BYTES + ty * ARB;                   // row ty (+16 r)
    const float *bs = reinterpret_cast<const float *>(sm + s * ST_BYTES + A_BYTES) + tx * 4;
#pragma unroll
    for (int q = 0; q < BK / 4; ++q) {
      float4 b[4][2];
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int h = 0; h < 2; ++h) b[k][h] = *reinterpret_cast<const float4 *>(bs + (4 * q + k) * TN + 64 * h);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const float4 a = *reinterpret_cast<const float4 *>(as + r * 16 * ARB + ((VAR & 4) ? ((q ^ sw) << 4) : (q << 4)));
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float *x = &acc[r][4 * h];
          fwb::relax2k(x[0], x[1], x[2], x[3], a.x, a.y, b[0][h], b[1][h]);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float *x = &acc[r][4 * h];
          fwb::relax2k(x[0], x[1], x[2], x[3], a.z, a.w, b[2][h], b[3][h]);
        }
      }
    }
    if (VAR & 2) continue;
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (tid == 0 && ch + NS < nch) {   // refill this stage once every warp has released it
      mbar_wait(&empty[s], (ch / NS) & 1);
      mbar_expect_tx(&full[s], TXB);
      tma_2d(sm + s * ST_BYTES, &mapA, kb + (ch + NS) * BK, i0, &full[s]);
      tma_2d(sm + s * ST_BYTES + A_BYTES, &mapB, j0, kb + (ch + NS) * BK, &full[s]);
    }
  }
  // epilogue (as the library's KEY mode)
  const int kgrp = kb & ~255;
  int kmax = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = i0 + ty + 16 * r;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int jb = j0 + 4 * tx + 64 * h;
      float4 *dp = reinterpret_cast<float4 *>(D + (int64_t)i * ld + jb);
      const float4 old = *dp;
      float4 nv = old;
      bool any = false;
      int pv[4];
      bool chg[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = jb + e;
        const float m = acc[r][4 * h + e];
        chg[e] = m < fwb::vget(old, e);
        pv[e] = 0;
        if (chg[e]) {
          any = true;
          float key = m;
          if (VAR & 1) {
            const int kk = (int)(m - (float)(j & 255)) & 255;
            key = m - (float)kk;
            kmax = max(kmax, __float_as_int(key));
            pv[e] = kgrp + kk;
          }
          fwb::vset(nv, e, key);
        }
      }
      if (any) {
        *dp = nv;
        if (VAR & 1) {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (chg[e]) P[(int64_t)i * ld + jb + e] = pv[e];
        }
      }
    }
  }
  if (VAR & 1) {
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    if (lane == 0 && kmax > 0) atomicMax(maxkey, kmax);
  }
}

static int make_map(CUtensorMap *m, float *D, int64_t n, int box_cols, int box_rows, CUtensorMapSwizzle sw) {
  cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};          // {cols (innermost), rows}
  cuuint64_t strides[1] = {(cuuint64_t)n * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, D, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("cuTensorMapEncodeTiled failed %d\n", (int)r); return 1; }
  return 0;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int64_t n = 16384;
  std::vector<float> init(n * n);
  uint64_t x = 88172645463325252ull;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      const int w = i == j ? 0 : 1 + (int)(x % 100);
      init[i * n + j] = (float)(w * 256 + (j & 255));
    }
  float *D, *D2; int32_t *P, *P2; int *mk;
  CK(cudaMalloc(&D, n * n * 4)); CK(cudaMalloc(&P, n * n * 4)); CK(cudaMalloc(&mk, 4));
  CK(cudaMalloc(&D2, n * n * 4)); CK(cudaMalloc(&P2, n * n * 4));
  const int kb = 128 * 50;
  CUtensorMap mA, mB;
  const int var0 = getenv("P3T_VAR") ? atoi(getenv("P3T_VAR")) : 1;
  if (make_map(&mA, D, n, (var0 & 8) ? A_W : BK, TM, (var0 & 4) ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE)) return 1;
  if (make_map(&mB, D, n, TN, BK, CU_TENSOR_MAP_SWIZZLE_NONE)) return 1;
  const int bytes = NS * ST_BYTES + 1024 + 64;
  const int var = getenv("P3T_VAR") ? atoi(getenv("P3T_VAR")) : 1;
  auto kern = var == 3 ? p3t<3> : var == 19 ? p3t<19> : var == 11 ? p3t<11> : var == 7 ? p3t<7> : var == 5 ? p3t<5> : p3t<1>;
  if ((var & 4) != (SWZ ? 4 : 0) && (var & 4)) { printf("build with -DSWZ=1 for VAR & 4\n"); }
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  cudaFuncAttributes fa; CK(cudaFuncGetAttributes(&fa, kern));
  int occ = 0; CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, bytes));
  // reference: the library kernel on the same launch
  auto lib = fwb::minplus_tile_kernel<float, 128, 128, fwb::MODE_KEY, false>;
  const int lbytes = fwb::TileShape<128, 128>::kBytes;
  CK(cudaFuncSetAttribute(lib, cudaFuncAttributeMaxDynamicSharedMemorySize, lbytes));
  cudaFuncAttributes fl; CK(cudaFuncGetAttributes(&fl, lib));
  fwb::TileArgs a{};
  a.ld = n; a.B = D2 + (int64_t)kb * n; a.ldb = n; a.kb = kb; a.Kd = 128;
  a.rows_lim = (int)n; a.cols_lim = (int)n;
  a.mr_lo[0] = kb; a.mr_hi[0] = kb + 128; a.mc_lo[0] = kb; a.mc_hi[0] = kb + 128;
  dim3 g(n / TN, n / TM);
  // correctness: both from the same input, compare D and P
  CK(cudaMemcpy(D, init.data(), n * n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(D2, init.data(), n * n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(P, 0xff, n * n * 4)); CK(cudaMemset(P2, 0xff, n * n * 4));
  kern<<<g, 256, bytes>>>(D, P, mA, mB, n, kb, mk);
  lib<<<g, 256, lbytes>>>(D2, P2, a, mk);
  CK(cudaDeviceSynchronize());
  {
    std::vector<float> h1(n * n), h2(n * n); std::vector<int32_t> q1(n * n), q2(n * n);
    CK(cudaMemcpy(h1.data(), D, n * n * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h2.data(), D2, n * n * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(q1.data(), P, n * n * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(q2.data(), P2, n * n * 4, cudaMemcpyDeviceToHost));
    int64_t bad = 0, changed = 0;
    for (int64_t e = 0; e < n * n; ++e) { bad += h1[e] != h2[e] || q1[e] != q2[e]; changed += h1[e] != init[e]; }
    printf("{\"check\": \"tma vs library kernel\", \"var\": %d, \"mismatches\": %lld, \"changed\": %lld}\n", var, (long long)bad, (long long)changed);
    fflush(stdout);
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 10;
  const int64_t tr = n / TM - 1, tc = n / TN - 1;
  const double relax = (double)tr * TM * tc * TN * 128;
  for (int pass = 0; pass < 2; ++pass) {
    for (int which = 0; which < 2; ++which) {
      CK(cudaMemcpy(D, init.data(), n * n * 4, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(D2, init.data(), n * n * 4, cudaMemcpyHostToDevice));
      auto launch = [&]() {
        if (which == 0) kern<<<g, 256, bytes>>>(D, P, mA, mB, n, kb, mk);
        else lib<<<g, 256, lbytes>>>(D2, P2, a, mk);
      };
      launch(); launch();
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
      printf("{\"variant\": \"%s\", \"regs\": %d, \"spill\": %d, \"occ\": %d, \"ms\": %.4f, \"relax_per_clk_sm_at_max_clock\": %.2f}\n",
             which == 0 ? (var == 1 ? "tma-3st-mbar" : var == 3 ? "tma-3st-1wait-sync" : var == 11 ? "tma-3st-1wait-sync-pad36" : var == 19 ? "tma-3st-1wait-sync-prefetch" : var == 7 ? "tma-3st-1wait-sync-swz" : "tma-3st-mbar-swz") : "library", which == 0 ? fa.numRegs : fl.numRegs,
             (int)(which == 0 ? fa.localSizeBytes : fl.localSizeBytes), which == 0 ? occ : 2, ms,
             relax / (ms * 1e-3) / (sms * (double)clk * 1e3));
      fflush(stdout);
    }
  }
  return 0;
}

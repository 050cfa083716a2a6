// Phase-3 tile-shape / schedule explorer (development tool, not part of the library).
// A parametric copy of the min-plus tile kernel: per-thread RM rows x 4H columns,
// TX x TY threads, MINB resident CTAs (register cap), BK-deep k chunks, NS stages.
// Times one phase-3 launch (n x n, K-depth 128) per variant on key-encoded integer data
// and prints relaxations / clock / SM at the max clock (the stated roofline is 64).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <vector>
#include "../fw_kernels.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ void cpa16(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cpc() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void cpw() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }


__device__ __forceinline__ float fadd_rn(float a, float b) {
  float r; asm("add.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r;
}
// relaxation variants: MODE 0 = FADD2 (production), 1 = scalar FADD, 2 = half FADD2 / half FADD
template <int M>
__device__ __forceinline__ void relax2v(float &x0, float &x1, float &x2, float &x3, float a0, float a1,
                                        const float4 &b0, const float4 &b1) {
  if (M == 0) {
    fwb::relax2k(x0, x1, x2, x3, a0, a1, b0, b1);
  } else if (M == 1) {
    x0 = fminf(x0, fminf(fadd_rn(a0, b0.x), fadd_rn(a1, b1.x)));
    x1 = fminf(x1, fminf(fadd_rn(a0, b0.y), fadd_rn(a1, b1.y)));
    x2 = fminf(x2, fminf(fadd_rn(a0, b0.z), fadd_rn(a1, b1.z)));
    x3 = fminf(x3, fminf(fadd_rn(a0, b0.w), fadd_rn(a1, b1.w)));
  } else {
    const float2 s0 = __fadd2_rn(make_float2(a0, a0), make_float2(b0.x, b0.y));
    const float2 s1 = __fadd2_rn(make_float2(a1, a1), make_float2(b1.x, b1.y));
    x0 = fminf(x0, fminf(s0.x, s1.x));
    x1 = fminf(x1, fminf(s0.y, s1.y));
    x2 = fminf(x2, fminf(fadd_rn(a0, b0.z), fadd_rn(a1, b1.z)));
    x3 = fminf(x3, fminf(fadd_rn(a0, b0.w), fadd_rn(a1, b1.w)));
  }
}

// VAR bits: 1 = key epilogue with P (else plain), 2 = L2 prefetch of the epilogue tile,
//           4 = k-outer order (all rows for k-pair 0 then k-pair 1 per q), 8 = no epilogue store
__device__ int g_kd = 128;   // k depth of one launch (128: one round; 256: a pair of rounds)
static int h_kd = 128;
template <int RM, int H, int TX, int TY, int MINB, int BK, int NS, int VAR>
__global__ void __launch_bounds__(TX * TY, MINB)
p3x(float *__restrict__ D, int32_t *__restrict__ P, int64_t ld, int kb, int *maxkey) {
  constexpr int NT = TX * TY, TM = RM * TY, TN = 4 * H * TX, AS = BK + 4;
  constexpr int SA = TM * AS, SB = BK * TN, ST = SA + SB;
  extern __shared__ __align__(16) float sm[];
  const int i0 = blockIdx.y * TM, j0 = blockIdx.x * TN;
  const int kd = g_kd;
  if ((i0 + TM > kb && i0 < kb + kd) || (j0 + TN > kb && j0 < kb + kd)) return;
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  if (VAR & 2) {
    constexpr int LPR = TN * 4 / 128;
    for (int l = tid; l < TM * LPR; l += NT)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(D + (int64_t)(i0 + l / LPR) * ld + j0 + (l % LPR) * 32));
  }
  constexpr int AC = TM * BK / 4, BC = BK * TN / 4;   // 16-B copies per chunk
  constexpr int A_PER = AC / NT, A_ROWS = NT / (BK / 4), B_PER = BC / NT, B_ROWS = NT / (TN / 4);
  static_assert(A_PER * NT == AC && B_PER * NT == BC && A_ROWS * (BK / 4) == NT && B_ROWS * (TN / 4) == NT, "copy map");
  const int a_r = tid / (BK / 4), a_c = (tid % (BK / 4)) * 4;
  const int b_r = tid / (TN / 4), b_c = (tid % (TN / 4)) * 4;
  const float *a_src = D + (int64_t)(i0 + a_r) * ld + kb + a_c;
  const float *b_src = D + (int64_t)(kb + b_r) * ld + j0 + b_c;
  const unsigned s_a = (unsigned)__cvta_generic_to_shared(sm + a_r * AS + a_c);
  const unsigned s_b = (unsigned)__cvta_generic_to_shared(sm + SA + b_r * TN + b_c);
  auto load = [&](int s, int k0) {
#pragma unroll
    for (int t = 0; t < A_PER; ++t)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s_a + (s * ST + t * A_ROWS * AS) * 4),
                   "l"(a_src + k0 + (int64_t)t * A_ROWS * ld) : "memory");
#pragma unroll
    for (int t = 0; t < B_PER; ++t)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s_b + (s * ST + t * B_ROWS * TN) * 4),
                   "l"(b_src + (int64_t)(k0 + t * B_ROWS) * ld) : "memory");
    cpc();
  };
  float acc[RM][4 * H];
#pragma unroll
  for (int r = 0; r < RM; ++r)
#pragma unroll
    for (int c = 0; c < 4 * H; ++c) acc[r][c] = __int_as_float(0x7f800000);
  const int nch = kd / BK;
#pragma unroll 1
  for (int s = 0; s < NS - 1; ++s) load(s, s * BK);
#pragma unroll 1
  if (VAR & 32) { cpw<0>(); __syncthreads(); }
#pragma unroll 1
  for (int ch = 0; ch < nch * ((VAR & 32) ? 8 : 1); ++ch) {
    if ((VAR & 1024) && NS >= 3) {   // 1024: wait, barrier, then issue chunk ch+NS-1 (one barrier per chunk)
      const int ahead = min(NS - 2, nch - 1 - ch);
      if (ahead >= 2) cpw<2>(); else if (ahead == 1) cpw<1>(); else cpw<0>();
      __syncthreads();
      if (ch + NS - 1 < nch) load((ch + NS - 1) % NS, (ch + NS - 1) * BK);
    } else if (!(VAR & 32)) {
      if (ch + NS - 1 < nch) { load((ch + NS - 1) % NS, (ch + NS - 1) * BK); cpw<NS - 1>(); }
      else {
        const int ahead = nch - 1 - ch;   // chunks already in flight beyond ch
        if (ahead >= 2) cpw<2>(); else if (ahead == 1) cpw<1>(); else cpw<0>();
      }
      __syncthreads();
    }
    if ((VAR & 256) && ch == nch - 1) {   // stage the epilogue's old-D lines into L1 (~1/4 tile ahead)
#pragma unroll
      for (int r = 0; r < RM; ++r)
#pragma unroll
        for (int h = 0; h < H; ++h)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(D + (int64_t)(i0 + ty + TY * r) * ld + j0 + 4 * tx + 4 * TX * h));
    }
    const float *as = sm + ((VAR & 32) ? 0 : (ch % NS)) * ST + ty * AS;
    const float *bs = sm + ((VAR & 32) ? 0 : (ch % NS)) * ST + SA + tx * 4;
#pragma unroll
    for (int q = 0; q < BK / 4; ++q) {
      if (VAR & 16) {   // b for one k-pair at a time (16 fewer live registers), float2 a loads
#pragma unroll
        for (int kp = 0; kp < 2; ++kp) {
          float4 b2[2][H];
#pragma unroll
          for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int h = 0; h < H; ++h) b2[k][h] = *reinterpret_cast<const float4 *>(bs + (4 * q + 2 * kp + k) * TN + 4 * TX * h);
#pragma unroll
          for (int r = 0; r < RM; ++r) {
            const float2 a = *reinterpret_cast<const float2 *>(as + TY * r * AS + 4 * q + 2 * kp);
#pragma unroll
            for (int h = 0; h < H; ++h) {
              float *x = &acc[r][4 * h];
              fwb::relax2k(x[0], x[1], x[2], x[3], a.x, a.y, b2[0][h], b2[1][h]);
            }
          }
        }
        continue;
      }
      float4 b[4][H];
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int h = 0; h < H; ++h) b[k][h] = *reinterpret_cast<const float4 *>(bs + (4 * q + k) * TN + 4 * TX * h);
      if (VAR & 12288) {   // 4096 / 8192: rows in groups of G = 4 / 2, per group k-pair outer, then
                           // column pair, then the G rows (mix_probe lds-G4: 78.0 vs 74.5)
        constexpr int G = (VAR & 4096) ? 4 : 2;
#pragma unroll
        for (int r = 0; r < RM; r += G) {
          float4 a[G];
#pragma unroll
          for (int g = 0; g < G; ++g) a[g] = *reinterpret_cast<const float4 *>(as + TY * (r + g) * AS + 4 * q);
#pragma unroll
          for (int kp = 0; kp < 2; ++kp)
#pragma unroll
            for (int h = 0; h < H; ++h)
#pragma unroll
              for (int pos = 0; pos < 2; ++pos) {
                const float4 bk = b[2 * kp][h], bk1 = b[2 * kp + 1][h];
                const float2 b0 = pos ? make_float2(bk.z, bk.w) : make_float2(bk.x, bk.y);
                const float2 b1 = pos ? make_float2(bk1.z, bk1.w) : make_float2(bk1.x, bk1.y);
                float2 s0[G], s1[G];
#pragma unroll
                for (int g = 0; g < G; ++g) {
                  const float a0 = kp ? a[g].z : a[g].x, a1 = kp ? a[g].w : a[g].y;
                  s0[g] = __fadd2_rn(make_float2(a0, a0), b0);
                  s1[g] = __fadd2_rn(make_float2(a1, a1), b1);
                }
#pragma unroll
                for (int g = 0; g < G; ++g) {
                  float *x = &acc[r + g][4 * h + 2 * pos];
                  x[0] = fminf(x[0], fminf(s0[g].x, s1[g].x));
                  x[1] = fminf(x[1], fminf(s0[g].y, s1[g].y));
                }
              }
        }
      } else if (VAR & 4) {
        float4 a[RM];
#pragma unroll
        for (int r = 0; r < RM; ++r) a[r] = *reinterpret_cast<const float4 *>(as + TY * r * AS + 4 * q);
#pragma unroll
        for (int kp = 0; kp < 2; ++kp)
#pragma unroll
          for (int r = 0; r < RM; ++r)
#pragma unroll
            for (int h = 0; h < H; ++h) {
              float *x = &acc[r][4 * h];
              fwb::relax2k(x[0], x[1], x[2], x[3], kp ? a[r].z : a[r].x, kp ? a[r].w : a[r].y,
                           b[2 * kp][h], b[2 * kp + 1][h]);
            }
      } else {
#pragma unroll
        for (int r = 0; r < RM; ++r) {
          const float4 a = *reinterpret_cast<const float4 *>(as + TY * r * AS + 4 * q);
          if (VAR & 2048) {   // scalar-reuse order: all FADD2 of a_k, then of a_k+1, then the FMNMX3s
#pragma unroll
            for (int kp = 0; kp < 2; ++kp) {
              const float a0 = kp ? a.z : a.x, a1 = kp ? a.w : a.y;
              float2 s0[H][2], s1[H][2];
#pragma unroll
              for (int h = 0; h < H; ++h) {
                s0[h][0] = __fadd2_rn(make_float2(a0, a0), make_float2(b[2 * kp][h].x, b[2 * kp][h].y));
                s0[h][1] = __fadd2_rn(make_float2(a0, a0), make_float2(b[2 * kp][h].z, b[2 * kp][h].w));
              }
#pragma unroll
              for (int h = 0; h < H; ++h) {
                s1[h][0] = __fadd2_rn(make_float2(a1, a1), make_float2(b[2 * kp + 1][h].x, b[2 * kp + 1][h].y));
                s1[h][1] = __fadd2_rn(make_float2(a1, a1), make_float2(b[2 * kp + 1][h].z, b[2 * kp + 1][h].w));
              }
#pragma unroll
              for (int h = 0; h < H; ++h) {
                float *x = &acc[r][4 * h];
                x[0] = fminf(x[0], fminf(s0[h][0].x, s1[h][0].x));
                x[1] = fminf(x[1], fminf(s0[h][0].y, s1[h][0].y));
                x[2] = fminf(x[2], fminf(s0[h][1].x, s1[h][1].x));
                x[3] = fminf(x[3], fminf(s0[h][1].y, s1[h][1].y));
              }
            }
            continue;
          }
#pragma unroll
          for (int h = 0; h < H; ++h) {
            float *x = &acc[r][4 * h];
            relax2v<(VAR >> 6) & 3>(x[0], x[1], x[2], x[3], a.x, a.y, b[0][h], b[1][h]);
          }
#pragma unroll
          for (int h = 0; h < H; ++h) {
            float *x = &acc[r][4 * h];
            relax2v<(VAR >> 6) & 3>(x[0], x[1], x[2], x[3], a.z, a.w, b[2][h], b[3][h]);
          }
        }
      }
    }
    if (!(VAR & 32) && !((VAR & (512 | 1024)) && NS >= 3)) __syncthreads();   // 512/1024: one barrier per chunk
    else asm volatile("" ::: "memory");
  }
  if (VAR & 8) {   // no epilogue: keep acc live
    float s = 0;
#pragma unroll
    for (int r = 0; r < RM; ++r)
#pragma unroll
      for (int c = 0; c < 4 * H; ++c) s = fminf(s, acc[r][c]);
    if (s < -1.f) D[tid] = s;
    return;
  }
  const int kgrp = kb & ~127;
  int kmax = 0;
#pragma unroll
  for (int r = 0; r < RM; ++r) {
    const int i = i0 + ty + TY * r;
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int jb = j0 + 4 * tx + 4 * TX * h;
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
            const int kk = (int)(m - (float)(j & 127)) & 127;
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
    if ((tid & 31) == 0 && kmax > 0) atomicMax(maxkey, kmax);
  }
}

static std::vector<float> g_init;

template <int RM, int H, int TX, int TY, int MINB, int BK, int NS, int VAR>
int run(const char *tag, float *D, int32_t *P, int *mk, int64_t n, int sms, int clk_khz) {
  constexpr int TM = RM * TY, TN = 4 * H * TX;
  const int bytes = NS * (TM * (BK + 4) + BK * TN) * 4;
  auto kern = p3x<RM, H, TX, TY, MINB, BK, NS, VAR>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, TX * TY, bytes));
  CK(cudaMemcpy(D, g_init.data(), n * n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpyToSymbol(g_kd, &h_kd, sizeof(int)));
  dim3 g(n / TN, n / TM);
  const int kb = 128 * 50;
  for (int w = 0; w < 2; ++w) kern<<<g, TX * TY, bytes>>>(D, P, n, kb, mk);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 10;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) kern<<<g, TX * TY, bytes>>>(D, P, n, kb, mk);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  // relaxations actually done: tiles outside the excluded strip (TM/TN-aligned exclusion)
  const int64_t tr = n / TM - (h_kd + TM - 1) / TM, tc = n / TN - (h_kd + TN - 1) / TN;
  const double relax = (double)tr * TM * tc * TN * h_kd * ((VAR & 32) ? 8 : 1);
  printf("{\"variant\": \"%s\", \"kd\": %d, \"RM\": %d, \"H\": %d, \"TX\": %d, \"TY\": %d, \"minb\": %d, \"BK\": %d, \"NS\": %d, \"var\": %d, "
         "\"regs\": %d, \"spill\": %d, \"occ\": %d, \"ms\": %.4f, \"relax_per_clk_sm_at_max_clock\": %.2f, \"tflops\": %.3f}\n",
         tag, h_kd, RM, H, TX, TY, MINB, BK, NS, VAR, fa.numRegs, (int)fa.localSizeBytes, occ, ms,
         relax / (ms * 1e-3) / (sms * (double)clk_khz * 1e3), 2 * relax / (ms * 1e-3) / 1e12);
  fflush(stdout);
  return 0;
}

// the library's stream kernel (KEY, 128 x 128) on the same launch
template <int MODE = fwb::MODE_KEY>
int runlib(const char *tag, float *D, int32_t *P, int *mk, int64_t n, int sms, int clk_khz) {
  auto lib = fwb::minplus_tile_kernel<float, 128, 128, MODE, false>;
  const int lbytes = fwb::TileShape<128, 128>::kBytes;
  CK(cudaFuncSetAttribute(lib, cudaFuncAttributeMaxDynamicSharedMemorySize, lbytes));
  cudaFuncAttributes fl; CK(cudaFuncGetAttributes(&fl, lib));
  const int kb = 128 * 50;
  fwb::TileArgs a{};
  a.ld = n; a.B = D + (int64_t)kb * n; a.ldb = n; a.kb = kb; a.Kd = h_kd;
  a.rows_lim = (int)n; a.cols_lim = (int)n; a.tag = kb / 128;
  a.mr_lo[0] = kb; a.mr_hi[0] = kb + h_kd; a.mc_lo[0] = kb; a.mc_hi[0] = kb + h_kd;
  CK(cudaMemcpy(D, g_init.data(), n * n * 4, cudaMemcpyHostToDevice));
  dim3 g(n / 128, n / 128);
  for (int w = 0; w < 2; ++w) lib<<<g, 256, lbytes>>>(D, P, a, mk);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 10;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) lib<<<g, 256, lbytes>>>(D, P, a, mk);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const int64_t t = n / 128 - h_kd / 128;
  const double relax = (double)t * 128 * t * 128 * h_kd;
  printf("{\"variant\": \"%s\", \"kd\": %d, \"regs\": %d, \"spill\": %d, \"ms\": %.4f, \"relax_per_clk_sm_at_max_clock\": %.2f, \"tflops\": %.3f}\n",
         tag, h_kd, fl.numRegs, (int)fl.localSizeBytes, ms, relax / (ms * 1e-3) / (sms * (double)clk_khz * 1e3), 2 * relax / (ms * 1e-3) / 1e12);
  fflush(stdout);
  return 0;
}


// k-pair variant: B comes from a packed copy of the pivot strip, Sp[k/2][j][2] =
// (B[k][j], B[k+1][j]); FADD2 adds the pair (a_ik, a_i,k+1) to (b_kj, b_k+1,j) and one
// FMNMX3 folds both candidates into x_ij: a 1:1 FADD2 -> FMNMX3 dependency.
// Thread owns rows ty + TY*r and column pairs 2tx + 2TX*c (c < CP).
template <int RM, int CP, int TX, int TY, int MINB, int BK, int NS, int VAR>
__global__ void __launch_bounds__(TX * TY, MINB)
p3k(float *__restrict__ D, int32_t *__restrict__ P, const float *__restrict__ Sp, int64_t ld, int kb, int *maxkey) {
  constexpr int NT = TX * TY, TM = RM * TY, TN = 2 * CP * TX, AS = BK + 4;
  constexpr int SA = TM * AS, SB = BK * TN, ST = SA + SB;
  extern __shared__ __align__(16) float sm[];
  const int i0 = blockIdx.y * TM, j0 = blockIdx.x * TN;
  if ((i0 + TM > kb && i0 < kb + 128) || (j0 + TN > kb && j0 < kb + 128)) return;
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  if (VAR & 2) {
    constexpr int LPR = TN * 4 / 128;
    for (int l = tid; l < TM * LPR; l += NT)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(D + (int64_t)(i0 + l / LPR) * ld + j0 + (l % LPR) * 32));
  }
  // A chunk: TM x BK row-major; B chunk: BK/2 packed rows of 2*TN floats
  constexpr int AC = TM * BK / 4, BC = BK * TN / 4;
  constexpr int A_PER = AC / NT, A_ROWS = NT / (BK / 4), B_PER = BC / NT, B_ROWS = NT / (2 * TN / 4);
  static_assert(A_PER * NT == AC && B_PER * NT == BC && A_ROWS * (BK / 4) == NT && B_ROWS * (2 * TN / 4) == NT, "copy map");
  const int a_r = tid / (BK / 4), a_c = (tid % (BK / 4)) * 4;
  const int b_r = tid / (2 * TN / 4), b_c = (tid % (2 * TN / 4)) * 4;
  const float *a_src = D + (int64_t)(i0 + a_r) * ld + kb + a_c;
  const float *b_src = Sp + (int64_t)(kb / 2 + b_r) * 2 * ld + 2 * j0 + b_c;
  const unsigned s_a = (unsigned)__cvta_generic_to_shared(sm + a_r * AS + a_c);
  const unsigned s_b = (unsigned)__cvta_generic_to_shared(sm + SA + b_r * 2 * TN + b_c);
  auto load = [&](int s, int k0) {
#pragma unroll
    for (int t = 0; t < A_PER; ++t)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s_a + (s * ST + t * A_ROWS * AS) * 4),
                   "l"(a_src + k0 + (int64_t)t * A_ROWS * ld) : "memory");
#pragma unroll
    for (int t = 0; t < B_PER; ++t)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s_b + (s * ST + t * B_ROWS * 2 * TN) * 4),
                   "l"(b_src + (int64_t)(k0 / 2 + t * B_ROWS) * 2 * ld) : "memory");
    cpc();
  };
  float acc[RM][2 * CP];
#pragma unroll
  for (int r = 0; r < RM; ++r)
#pragma unroll
    for (int c = 0; c < 2 * CP; ++c) acc[r][c] = __int_as_float(0x7f800000);
  constexpr int nch = 128 / BK;
#pragma unroll 1
  for (int s = 0; s < NS - 1; ++s) load(s, s * BK);
#pragma unroll 1
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + NS - 1 < nch) { load((ch + NS - 1) % NS, (ch + NS - 1) * BK); cpw<NS - 1>(); }
    else if (NS == 3 && ch + 1 < nch) cpw<1>();
    else cpw<0>();
    __syncthreads();
    const float *as = sm + (ch % NS) * ST + ty * AS;
    const float *bs = sm + (ch % NS) * ST + SA + tx * 4;
#pragma unroll
    for (int q = 0; q < BK / 4; ++q) {
      float4 b[2][CP];   // b[kp][c] = (B[k][j], B[k+1][j], B[k][j+1], B[k+1][j+1]), k = 4q + 2kp
#pragma unroll
      for (int kp = 0; kp < 2; ++kp)
#pragma unroll
        for (int c = 0; c < CP; ++c) b[kp][c] = *reinterpret_cast<const float4 *>(bs + (2 * q + kp) * 2 * TN + 4 * TX * c);
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        const float4 a = *reinterpret_cast<const float4 *>(as + TY * r * AS + 4 * q);
#pragma unroll
        for (int kp = 0; kp < 2; ++kp) {
          const float2 ap = kp ? make_float2(a.z, a.w) : make_float2(a.x, a.y);
#pragma unroll
          for (int c = 0; c < CP; ++c) {
            const float2 s0 = __fadd2_rn(ap, make_float2(b[kp][c].x, b[kp][c].y));
            const float2 s1 = __fadd2_rn(ap, make_float2(b[kp][c].z, b[kp][c].w));
            acc[r][2 * c] = fminf(acc[r][2 * c], fminf(s0.x, s0.y));
            acc[r][2 * c + 1] = fminf(acc[r][2 * c + 1], fminf(s1.x, s1.y));
          }
        }
      }
    }
    __syncthreads();
  }
  if (VAR & 8) {
    float s = 0;
#pragma unroll
    for (int r = 0; r < RM; ++r)
#pragma unroll
      for (int c = 0; c < 2 * CP; ++c) s = fminf(s, acc[r][c]);
    if (s < -1.f) D[tid] = s;
    return;
  }
  const int kgrp = kb & ~127;
  int kmax = 0;
#pragma unroll
  for (int r = 0; r < RM; ++r) {
    const int i = i0 + ty + TY * r;
#pragma unroll
    for (int c = 0; c < CP; ++c) {
      const int jb = j0 + 2 * tx + 2 * TX * c;
      float2 *dp = reinterpret_cast<float2 *>(D + (int64_t)i * ld + jb);
      const float2 old = *dp;
      float2 nv = old;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = jb + e;
        const float m = acc[r][2 * c + e];
        const float o = e ? old.y : old.x;
        if (m < o) {
          float key = m;
          if (VAR & 1) {
            const int kk = (int)(m - (float)(j & 127)) & 127;
            key = m - (float)kk;
            kmax = max(kmax, __float_as_int(key));
            P[(int64_t)i * ld + j] = kgrp + kk;
          }
          if (e) nv.y = key; else nv.x = key;
        }
      }
      if (nv.x != old.x || nv.y != old.y) *dp = nv;
    }
  }
  if (VAR & 1) {
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    if ((tid & 31) == 0 && kmax > 0) atomicMax(maxkey, kmax);
  }
}

template <int RM, int CP, int TX, int TY, int MINB, int BK, int NS, int VAR>
int runk(const char *tag, float *D, int32_t *P, const float *Sp, int *mk, int64_t n, int sms, int clk_khz) {
  constexpr int TM = RM * TY, TN = 2 * CP * TX;
  const int bytes = NS * (TM * (BK + 4) + BK * TN) * 4;
  auto kern = p3k<RM, CP, TX, TY, MINB, BK, NS, VAR>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, TX * TY, bytes));
  CK(cudaMemcpy(D, g_init.data(), n * n * 4, cudaMemcpyHostToDevice));
  dim3 g(n / TN, n / TM);
  const int kb = 128 * 50;
  for (int w = 0; w < 2; ++w) kern<<<g, TX * TY, bytes>>>(D, P, Sp, n, kb, mk);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 10;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) kern<<<g, TX * TY, bytes>>>(D, P, Sp, n, kb, mk);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const int64_t tr = n / TM - (128 + TM - 1) / TM, tc = n / TN - (128 + TN - 1) / TN;
  const double relax = (double)tr * TM * tc * TN * 128;
  printf("{\"variant\": \"%s\", \"RM\": %d, \"CP\": %d, \"TX\": %d, \"TY\": %d, \"minb\": %d, \"BK\": %d, \"NS\": %d, \"var\": %d, "
         "\"regs\": %d, \"spill\": %d, \"occ\": %d, \"ms\": %.4f, \"relax_per_clk_sm_at_max_clock\": %.2f, \"tflops\": %.3f}\n",
         tag, RM, CP, TX, TY, MINB, BK, NS, VAR, fa.numRegs, (int)fa.localSizeBytes, occ, ms,
         relax / (ms * 1e-3) / (sms * (double)clk_khz * 1e3), 2 * relax / (ms * 1e-3) / 1e12);
  fflush(stdout);
  return 0;
}


__device__ int g_smslot[256];
__device__ long long g_stagger_clk;
// Persistent variant of the 3-stage / one-barrier 8x8 kernel: grid = 2 CTAs per SM, each CTA
// walks tiles blockIdx.x, blockIdx.x + gridDim.x, ... and the cp.async chunk stream runs across
// tile boundaries (the next tile's first chunks load during this tile's last chunk + epilogue).
template <int VAR>
__global__ void __launch_bounds__(256, 2)
p3p(float *__restrict__ D, int32_t *__restrict__ P, int64_t ld, int kb, int *maxkey, int tiles) {
  constexpr int TM = 128, TN = 128, BK = 32, NS = 3, AS = BK + 4, SA = TM * AS, SB = BK * TN, ST = SA + SB;
  constexpr int NCH = 128 / BK, RM = 8, H = 2, TX = 16, TY = 16;
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  const int tk = kb / 128, ntc = tiles - 1;                 // tiles per dim; one excluded
  const int my = (ntc * ntc - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;   // my tile count
  const int total = my * NCH;
  auto origin = [&](int i, int &i0, int &j0) {
    const int t = blockIdx.x + i * gridDim.x;
    int by = t / ntc, bx = t % ntc;
    by += by >= tk;
    bx += bx >= tk;
    i0 = by * TM;
    j0 = bx * TN;
  };
  const int a_r = tid / (BK / 4), a_c = (tid % (BK / 4)) * 4;
  const int b_r = tid / (TN / 4), b_c = (tid % (TN / 4)) * 4;
  const unsigned s_a = (unsigned)__cvta_generic_to_shared(sm + a_r * AS + a_c);
  const unsigned s_b = (unsigned)__cvta_generic_to_shared(sm + SA + b_r * TN + b_c);
  auto load = [&](int gch) {
    int i0, j0;
    origin(gch / NCH, i0, j0);
    const int k0 = (gch % NCH) * BK, s = gch % NS;
    const float *a_src = D + (int64_t)(i0 + a_r) * ld + kb + a_c + k0;
    const float *b_src = D + (int64_t)(kb + k0 + b_r) * ld + j0 + b_c;
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s_a + (s * ST + t * 32 * AS) * 4),
                   "l"(a_src + (int64_t)t * 32 * ld) : "memory");
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s_b + (s * ST + t * 8 * TN) * 4),
                   "l"(b_src + (int64_t)t * 8 * ld) : "memory");
    cpc();
  };
  float acc[RM][4 * H];
  if (VAR & 4) {
    // staggered start: the second CTA to arrive on an SM waits about half a tile, so the two
    // co-resident CTAs stop running their epilogues (and the next tile's pipeline fill) in lock-step
    __shared__ int slot;
    if (tid == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      slot = atomicAdd(g_smslot + smid, 1) & 1;
    }
    __syncthreads();
    if (slot) {
      const long long t0 = clock64();
      while (clock64() - t0 < g_stagger_clk) __nanosleep(1000);
    }
  }
  if (total > 0) load(0);
  if (total > 1) load(1);
#pragma unroll 1
  for (int gch = 0; gch < total; ++gch) {
    if (gch + 1 < total) cpw<1>(); else cpw<0>();
    __syncthreads();
    if (gch + 2 < total) load(gch + 2);
    const int ch = gch % NCH;
    if (ch == 0) {
#pragma unroll
      for (int r = 0; r < RM; ++r)
#pragma unroll
        for (int c = 0; c < 4 * H; ++c) acc[r][c] = __int_as_float(0x7f800000);
      if (VAR & 2) {
        int i0, j0;
        origin(gch / NCH, i0, j0);
        for (int l = tid; l < TM * 4; l += 256)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(D + (int64_t)(i0 + l / 4) * ld + j0 + (l % 4) * 32));
      }
    }
    const float *as = sm + (gch % NS) * ST + ty * AS;
    const float *bs = sm + (gch % NS) * ST + SA + tx * 4;
#pragma unroll
    for (int q = 0; q < BK / 4; ++q) {
      float4 b[4][H];
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int h = 0; h < H; ++h) b[k][h] = *reinterpret_cast<const float4 *>(bs + (4 * q + k) * TN + 4 * TX * h);
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        const float4 a = *reinterpret_cast<const float4 *>(as + TY * r * AS + 4 * q);
#pragma unroll
        for (int h = 0; h < H; ++h) {
          float *x = &acc[r][4 * h];
          fwb::relax2k(x[0], x[1], x[2], x[3], a.x, a.y, b[0][h], b[1][h]);
        }
#pragma unroll
        for (int h = 0; h < H; ++h) {
          float *x = &acc[r][4 * h];
          fwb::relax2k(x[0], x[1], x[2], x[3], a.z, a.w, b[2][h], b[3][h]);
        }
      }
    }
    if (ch == NCH - 1) {   // epilogue of this tile (keyed, as the library's)
      int i0, j0;
      origin(gch / NCH, i0, j0);
      const int kgrp = kb & ~127;
      int kmax = 0;
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        const int i = i0 + ty + TY * r;
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const int jb = j0 + 4 * tx + 4 * TX * h;
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
              const int kk = (int)(m - (float)(j & 127)) & 127;
              const float key = m - (float)kk;
              kmax = max(kmax, __float_as_int(key));
              pv[e] = kgrp + kk;
              fwb::vset(nv, e, key);
            }
          }
          if (any) {
            *dp = nv;
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (chg[e]) P[(int64_t)i * ld + jb + e] = pv[e];
          }
        }
      }
      kmax = __reduce_max_sync(0xffffffffu, kmax);
      if ((tid & 31) == 0 && kmax > 0) atomicMax(maxkey, kmax);
    }
  }
}

static long long g_stagger = 0;
template <int VAR>
int runp(const char *tag, float *D, int32_t *P, int *mk, int64_t n, int sms, int clk_khz, int per_sm) {
  const int bytes = 3 * (128 * 36 + 32 * 128) * 4;
  auto kern = p3p<VAR>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kern));
  CK(cudaMemcpy(D, g_init.data(), n * n * 4, cudaMemcpyHostToDevice));
  const int tiles = (int)(n / 128), kb = 128 * 50;
  const int grid = sms * per_sm;
  CK(cudaMemcpyToSymbol(g_stagger_clk, &g_stagger, sizeof(long long)));
  for (int w = 0; w < 2; ++w) kern<<<grid, 256, bytes>>>(D, P, n, kb, mk, tiles);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 10;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) kern<<<grid, 256, bytes>>>(D, P, n, kb, mk, tiles);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const double relax = (double)(tiles - 1) * 128 * (tiles - 1) * 128 * 128;
  printf("{\"variant\": \"%s\", \"RM\": 8, \"H\": 2, \"TX\": 16, \"TY\": 16, \"minb\": 2, \"BK\": 32, \"NS\": 3, \"var\": %d, "
         "\"regs\": %d, \"spill\": %d, \"occ\": %d, \"ms\": %.4f, \"relax_per_clk_sm_at_max_clock\": %.2f, \"tflops\": %.3f}\n",
         tag, VAR, fa.numRegs, (int)fa.localSizeBytes, per_sm, ms,
         relax / (ms * 1e-3) / (sms * (double)clk_khz * 1e3), 2 * relax / (ms * 1e-3) / 1e12);
  fflush(stdout);
  return 0;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int64_t n = 16384;
  g_init.resize(n * n);
  uint64_t x = 88172645463325252ull;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      const int w = i == j ? 0 : 1 + (int)(x % 100);
      g_init[i * n + j] = (float)(w * 128 + (j & 127));
    }
  float *D; int32_t *P; int *mk;
  CK(cudaMalloc(&D, n * n * 4)); CK(cudaMalloc(&P, n * n * 4)); CK(cudaMalloc(&mk, 4));
  // packed pivot strip Sp[k/2][j][2] (what phase 2 would write)
  float *Sp; CK(cudaMalloc(&Sp, n * n * 4));
  {
    std::vector<float> sp(n * n);
    for (int64_t k = 0; k < n; k += 2)
      for (int64_t j = 0; j < n; ++j) { sp[(k / 2) * 2 * n + 2 * j] = g_init[k * n + j]; sp[(k / 2) * 2 * n + 2 * j + 1] = g_init[(k + 1) * n + j]; }
    CK(cudaMemcpy(Sp, sp.data(), n * n * 4, cudaMemcpyHostToDevice));
  }
  for (int kd = 128; kd <= 256; kd += 128) {
    h_kd = kd;
    runlib("library-key", D, P, mk, n, sms, clk);
    run<8, 2, 16, 16, 2, 32, 3, 1024 + 3>("3st-1bar", D, P, mk, n, sms, clk);
    run<8, 2, 16, 16, 2, 32, 3, 1024 + 3 + 4>("3st-1bar-kouter", D, P, mk, n, sms, clk);
    run<8, 2, 16, 16, 2, 32, 3, 1024 + 3 + 4096>("3st-1bar-G4", D, P, mk, n, sms, clk);
    runlib("library-key-again", D, P, mk, n, sms, clk);
    // four CTAs of 128 threads per SM (same registers, 16 warps): 8 x 8 per thread, 128 x 64 tiles
    run<8, 2, 8, 16, 4, 16, 3, 1024 + 3>("4cta-128thr-128x64-bk16-3st", D, P, mk, n, sms, clk);
    run<8, 2, 8, 16, 4, 16, 4, 1024 + 3>("4cta-128thr-128x64-bk16-4st", D, P, mk, n, sms, clk);
    run<8, 2, 8, 16, 4, 16, 4, 1024 + 3 + 4>("4cta-128thr-128x64-bk16-4st-kouter", D, P, mk, n, sms, clk);
    // three CTAs per SM (24 warps): 4 x 8 per thread, 64 x 128 tiles
    runlib<fwb::MODE_TAG>("library-tag", D, P, mk, n, sms, clk);
    runlib<fwb::MODE_PLAIN>("library-plain", D, P, mk, n, sms, clk);
    // one CTA of 512 threads per SM (same registers per SM): 256 x 128 and 128 x 256 tiles
  }
  return 0;
}

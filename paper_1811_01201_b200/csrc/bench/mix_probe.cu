// Scheduling probe (development tool): the phase-3 relaxation pattern (FADD2 with a broadcast
// scalar + FMNMX3 folding two k into an accumulator) from registers only, asm volatile so
// nothing is hoisted, at several accumulator counts / warps per SM. Separates the instruction
// mix + occupancy limit from shared-memory loads, barriers and the epilogue.
#include <cuda_runtime.h>
#include <stdio.h>

__device__ __forceinline__ unsigned long long fadd2b(float a, unsigned long long b) {
  unsigned long long r;
  // a broadcast into both lanes: {a, a} + b
  asm volatile("{ .reg .b64 t; mov.b64 t, {%1, %1}; add.rn.f32x2 %0, t, %2; }" : "=l"(r) : "f"(a), "l"(b));
  return r;
}
__device__ __forceinline__ void min3v(float &x, float p, float q) {
  asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(x) : "f"(p), "f"(q));
}
__device__ __forceinline__ float lo(unsigned long long v) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return a; }
__device__ __forceinline__ float hi(unsigned long long v) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return b; }

// NA accumulators = RM rows x 8 columns; per iteration each accumulator gets 2 k (4 relax2k
// groups per row): 2*NA relaxations, NA FADD2 + NA FMNMX3.
template <int RM, int MINB, int ORDER>
__global__ void __launch_bounds__(256, MINB) probe(float *out, int iters, float seed) {
  constexpr int NA = RM * 8;
  float x[NA];
  float a[2 * RM];
  unsigned long long b[8];
#pragma unroll
  for (int i = 0; i < NA; ++i) x[i] = 1e30f;
#pragma unroll
  for (int i = 0; i < 2 * RM; ++i) a[i] = seed * (threadIdx.x + i);
#pragma unroll
  for (int i = 0; i < 8; ++i) { float p = seed + i, q = seed - i; asm("mov.b64 %0, {%1,%2};" : "=l"(b[i]) : "f"(p), "f"(q)); }
  unsigned long long zero;
  { float z0 = 0.f; asm("mov.b64 %0, {%1,%1};" : "=l"(zero) : "f"(z0)); }
  const unsigned wmask = reinterpret_cast<const unsigned *>(out)[4095];   // all ones at run time, opaque to ptxas
  for (int it = 0; it < iters; ++it) {
    // loop-carried B operands (b + 0, not foldable because of signed zero): without this
    // ptxas CSEs the FADD2s across iterations (8 extra FADD2 per 8*RM, not counted)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(b[i]) : "l"(zero));
    const int mrun = (int)wmask - it;   // never in [0, 64): wmask is all ones at run time
#pragma unroll
    for (int r = 0; r < RM; ++r) {
      if (ORDER == 6) {   // boustrophedon: a_k, a_k+1 | a_k+1, a_k | a_k, ... so every second FADD2 shares its scalar
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const unsigned long long s0 = fadd2b(a[2 * r], b[4 * h + 0]);
          const unsigned long long s1 = fadd2b(a[2 * r + 1], b[4 * h + 1]);
          float *xx = &x[8 * r + 4 * h];
          min3v(xx[0], lo(s0), lo(s1));
          min3v(xx[1], hi(s0), hi(s1));
          const unsigned long long s3 = fadd2b(a[2 * r + 1], b[4 * h + 3]);
          const unsigned long long s2 = fadd2b(a[2 * r], b[4 * h + 2]);
          min3v(xx[2], lo(s2), lo(s3));
          min3v(xx[3], hi(s2), hi(s3));
        }
      } else if (ORDER == 5) {   // cross variant (NOT min-plus): production FADD2 form, but each FMNMX3 reads
                          // the two halves of ONE result pair — isolates the FMNMX3 operand layout
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const unsigned long long s0 = fadd2b(a[2 * r], b[4 * h + 0]);
          const unsigned long long s1 = fadd2b(a[2 * r + 1], b[4 * h + 1]);
          const unsigned long long s2 = fadd2b(a[2 * r], b[4 * h + 2]);
          const unsigned long long s3 = fadd2b(a[2 * r + 1], b[4 * h + 3]);
          float *xx = &x[8 * r + 4 * h];
          min3v(xx[0], lo(s0), hi(s0));
          min3v(xx[1], lo(s1), hi(s1));
          min3v(xx[2], lo(s2), hi(s2));
          min3v(xx[3], lo(s3), hi(s3));
        }
      } else if (ORDER == 3) {   // scalar-pair order: both FADD2s of a_k, then both of a_k+1 (the scalar is reusable)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const unsigned long long s0 = fadd2b(a[2 * r], b[4 * h + 0]);
          const unsigned long long s2 = fadd2b(a[2 * r], b[4 * h + 2]);
          const unsigned long long s1 = fadd2b(a[2 * r + 1], b[4 * h + 1]);
          const unsigned long long s3 = fadd2b(a[2 * r + 1], b[4 * h + 3]);
          float *xx = &x[8 * r + 4 * h];
          min3v(xx[0], lo(s0), lo(s1));
          min3v(xx[1], hi(s0), hi(s1));
          min3v(xx[2], lo(s2), lo(s3));
          min3v(xx[3], hi(s2), hi(s3));
        }
      } else if (ORDER == 0) {   // production order: per 4 columns: 4 FADD2 then 4 FMNMX3
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const unsigned long long s0 = fadd2b(a[2 * r], b[4 * h + 0]);
          const unsigned long long s1 = fadd2b(a[2 * r + 1], b[4 * h + 1]);
          const unsigned long long s2 = fadd2b(a[2 * r], b[4 * h + 2]);
          const unsigned long long s3 = fadd2b(a[2 * r + 1], b[4 * h + 3]);
          float *xx = &x[8 * r + 4 * h];
          min3v(xx[0], lo(s0), lo(s1));
          min3v(xx[1], hi(s0), hi(s1));
          min3v(xx[2], lo(s2), lo(s3));
          min3v(xx[3], hi(s2), hi(s3));
        }
      } else if (ORDER >= 64) {
        // forced runs with a REAL basic-block boundary (session 5): a never-taken branch on a value
        // that changes every iteration (ISETP + BRA) between the FADD2 run (consecutive FADD2s share
        // the 64-bit b operand: .reuse) and the FMNMX3 run, so ptxas cannot interleave them
        constexpr int G = (ORDER & 15) ? (ORDER & 15) : 1;
        if (r % G == 0) {
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            const int b0 = 4 * (p / 2) + 2 * (p % 2), b1 = b0 + 1;
            unsigned long long s0[G], s1[G];
#pragma unroll
            for (int g = 0; g < G; ++g) s0[g] = fadd2b(a[2 * (r + g)], b[b0]);
#pragma unroll
            for (int g = 0; g < G; ++g) s1[g] = fadd2b(a[2 * (r + g) + 1], b[b1]);
            if (mrun == 2 * (r * 4 + p)) asm volatile("trap;");
#pragma unroll
            for (int g = 0; g < G; ++g) {
              min3v(x[8 * (r + g) + 2 * p], lo(s0[g]), lo(s1[g]));
              min3v(x[8 * (r + g) + 2 * p + 1], hi(s0[g]), hi(s1[g]));
            }
            if (mrun == 2 * (r * 4 + p) + 1) asm volatile("trap;");
          }
        }
      } else if (ORDER >= 16) {
        // forced runs (session 5): G rows; a scheduling fence between the FADD2 run (consecutive
        // FADD2s share the 64-bit b operand) and the FMNMX3 run, so ptxas cannot interleave them.
        // ORDER 16+G: bar.warp.sync as the fence; ORDER 32+G: a never-taken branch on a kernel argument
        constexpr int G = (ORDER & 15) ? (ORDER & 15) : 1;
        if (r % G == 0) {
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            const int b0 = 4 * (p / 2) + 2 * (p % 2), b1 = b0 + 1;
            unsigned long long s0[G], s1[G];
#pragma unroll
            for (int g = 0; g < G; ++g) s0[g] = fadd2b(a[2 * (r + g)], b[b0]);
#pragma unroll
            for (int g = 0; g < G; ++g) s1[g] = fadd2b(a[2 * (r + g) + 1], b[b1]);
            asm volatile("bar.warp.sync %0;" ::"r"(wmask) : "memory");
#pragma unroll
            for (int g = 0; g < G; ++g) {
              min3v(x[8 * (r + g) + 2 * p], lo(s0[g]), lo(s1[g]));
              min3v(x[8 * (r + g) + 2 * p + 1], hi(s0[g]), hi(s1[g]));
            }
            if (!(ORDER & 32)) asm volatile("bar.warp.sync %0;" ::"r"(wmask) : "memory");
          }
        }
      } else if (ORDER >= 2) {
        // b-pair reuse order (session 5): G = ORDER rows at a time; consecutive FADD2s share
        // the 64-bit b operand (same slot) and differ in the broadcast scalar a
        constexpr int G = ORDER >= 2 ? ORDER : 1;
        if (r % G == 0) {
#pragma unroll
          for (int p = 0; p < 4; ++p) {     // column pair p of the 8 columns
            const int b0 = 4 * (p / 2) + 2 * (p % 2), b1 = b0 + 1;
            unsigned long long s0[G], s1[G];
#pragma unroll
            for (int g = 0; g < G; ++g) s0[g] = fadd2b(a[2 * (r + g)], b[b0]);
#pragma unroll
            for (int g = 0; g < G; ++g) s1[g] = fadd2b(a[2 * (r + g) + 1], b[b1]);
#pragma unroll
            for (int g = 0; g < G; ++g) {
              min3v(x[8 * (r + g) + 2 * p], lo(s0[g]), lo(s1[g]));
              min3v(x[8 * (r + g) + 2 * p + 1], hi(s0[g]), hi(s1[g]));
            }
          }
        }
      } else {            // interleaved: FADD2 pair, FMNMX3 pair of the previous group
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const unsigned long long s0 = fadd2b(a[2 * r], b[4 * h + 0]);
          const unsigned long long s1 = fadd2b(a[2 * r + 1], b[4 * h + 1]);
          float *xx = &x[8 * r + 4 * h];
          min3v(xx[0], lo(s0), lo(s1));
          const unsigned long long s2 = fadd2b(a[2 * r], b[4 * h + 2]);
          min3v(xx[1], hi(s0), hi(s1));
          const unsigned long long s3 = fadd2b(a[2 * r + 1], b[4 * h + 3]);
          min3v(xx[2], lo(s2), lo(s3));
          min3v(xx[3], hi(s2), hi(s3));
        }
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NA; ++i) s += x[i];
  if (s == 1.2345f) out[threadIdx.x] = s;
}

template <int RM, int MINB, int ORDER>
void run(const char *tag, float *out, int sms, int clk) {
  const int iters = 4000;
  const int blocks = sms * MINB * 8;
  probe<RM, MINB, ORDER><<<blocks, 256>>>(out, 10, 1.0001f);
  cudaDeviceSynchronize();
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, probe<RM, MINB, ORDER>);
  int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, probe<RM, MINB, ORDER>, 256, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<RM, MINB, ORDER><<<blocks, 256>>>(out, iters, 1.0001f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double relax = (double)blocks * 256 * iters * RM * 8 * 2;
  printf("{\"probe\": \"%s\", \"RM\": %d, \"minb\": %d, \"order\": %d, \"regs\": %d, \"spill\": %d, \"occ\": %d, \"ms\": %.3f, \"relax_per_clk_sm_at_max\": %.2f, \"err\": \"%s\"}\n",
         tag, RM, MINB, ORDER, fa.numRegs, (int)fa.localSizeBytes, occ, ms, relax / (ms * 1e-3) / (sms * (double)clk * 1e3),
         cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}


// Production inner loop fed from shared memory: per q (4 k) 8 LDS.128 of B + per row one
// LDS.128 of A, relax2k as in fw_kernels.cuh; optional barrier every BAR q-steps.
// Addresses rotate with the iteration so nothing is loop-invariant.
template <int BAR, int MINB>
__global__ void __launch_bounds__(256, MINB) probe_lds(float *out, int iters) {
  constexpr int AS = 36, TN = 128;
  __shared__ __align__(16) float as_[128 * AS];
  __shared__ __align__(16) float bs_[32 * TN + 4];
  for (int e = threadIdx.x; e < 128 * AS; e += 256) as_[e] = 1.0f + (e % 97);
  for (int e = threadIdx.x; e < 32 * TN + 4; e += 256) bs_[e] = 2.0f + (e % 89);
  __syncthreads();
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 1e30f;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const int st = (it & 1) * 4;   // iteration-dependent addresses (inside the padding)
    const float *as = as_ + ty * AS + st;
    const float *bs = bs_ + tx * 4 + st;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 b[4][2];
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int h = 0; h < 2; ++h) b[k][h] = *reinterpret_cast<const float4 *>(bs + (4 * q + k) * TN + 64 * h);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const float4 a = *reinterpret_cast<const float4 *>(as + 16 * r * AS + 4 * q);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float *x = &acc[r][4 * h];
          const float2 s0 = __fadd2_rn(make_float2(a.x, a.x), make_float2(b[0][h].x, b[0][h].y));
          const float2 s1 = __fadd2_rn(make_float2(a.y, a.y), make_float2(b[1][h].x, b[1][h].y));
          const float2 s2 = __fadd2_rn(make_float2(a.x, a.x), make_float2(b[0][h].z, b[0][h].w));
          const float2 s3 = __fadd2_rn(make_float2(a.y, a.y), make_float2(b[1][h].z, b[1][h].w));
          x[0] = fminf(x[0], fminf(s0.x, s1.x)); x[1] = fminf(x[1], fminf(s0.y, s1.y));
          x[2] = fminf(x[2], fminf(s2.x, s3.x)); x[3] = fminf(x[3], fminf(s2.y, s3.y));
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float *x = &acc[r][4 * h];
          const float2 s0 = __fadd2_rn(make_float2(a.z, a.z), make_float2(b[2][h].x, b[2][h].y));
          const float2 s1 = __fadd2_rn(make_float2(a.w, a.w), make_float2(b[3][h].x, b[3][h].y));
          const float2 s2 = __fadd2_rn(make_float2(a.z, a.z), make_float2(b[2][h].z, b[2][h].w));
          const float2 s3 = __fadd2_rn(make_float2(a.w, a.w), make_float2(b[3][h].z, b[3][h].w));
          x[0] = fminf(x[0], fminf(s0.x, s1.x)); x[1] = fminf(x[1], fminf(s0.y, s1.y));
          x[2] = fminf(x[2], fminf(s2.x, s3.x)); x[3] = fminf(x[3], fminf(s2.y, s3.y));
        }
      }
    }
    if (BAR) __syncthreads();
  }
  float s = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[r][c];
  if (s == 1.2345f) out[threadIdx.x] = s;
}

template <int BAR, int MINB>
void run_lds(const char *tag, float *out, int sms, int clk) {
  const int iters = 400;
  const int blocks = sms * 2 * 8;
  probe_lds<BAR, MINB><<<blocks, 256>>>(out, 4);
  cudaDeviceSynchronize();
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, probe_lds<BAR, MINB>);
  int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, probe_lds<BAR, MINB>, 256, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe_lds<BAR, MINB><<<blocks, 256>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double relax = (double)blocks * 256 * iters * 64 * 32;
  printf("{\"probe\": \"%s\", \"bar\": %d, \"minb\": %d, \"regs\": %d, \"spill\": %d, \"occ\": %d, \"ms\": %.3f, \"relax_per_clk_sm_at_max\": %.2f, \"err\": \"%s\"}\n",
         tag, BAR, MINB, fa.numRegs, (int)fa.localSizeBytes, occ, ms, relax / (ms * 1e-3) / (sms * (double)clk * 1e3),
         cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

template <int BAR, int MINB, int G>
__global__ void __launch_bounds__(256, MINB) probe_lds_g(float *out, int iters) {
  constexpr int AS = 36, TN = 128;
  __shared__ __align__(16) float as_[128 * AS];
  __shared__ __align__(16) float bs_[32 * TN + 4];
  for (int e = threadIdx.x; e < 128 * AS; e += 256) as_[e] = 1.0f + (e % 97);
  for (int e = threadIdx.x; e < 32 * TN + 4; e += 256) bs_[e] = 2.0f + (e % 89);
  __syncthreads();
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 1e30f;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const int st = (it & 1) * 4;   // iteration-dependent addresses (inside the padding)
    const float *as = as_ + ty * AS + st;
    const float *bs = bs_ + tx * 4 + st;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 b[4][2];
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int h = 0; h < 2; ++h) b[k][h] = *reinterpret_cast<const float4 *>(bs + (4 * q + k) * TN + 64 * h);
#pragma unroll
      for (int r = 0; r < 8; r += G) {
        float4 a[G];
#pragma unroll
        for (int g = 0; g < G; ++g) a[g] = *reinterpret_cast<const float4 *>(as + 16 * (r + g) * AS + 4 * q);
#pragma unroll
        for (int kp = 0; kp < 2; ++kp)
#pragma unroll
          for (int h = 0; h < 2; ++h)
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
    }
    if (BAR) __syncthreads();
  }
  float s = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[r][c];
  if (s == 1.2345f) out[threadIdx.x] = s;
}

template <int BAR, int MINB, int G>
void run_lds_g(const char *tag, float *out, int sms, int clk) {
  const int iters = 400;
  const int blocks = sms * 2 * 8;
  probe_lds_g<BAR, MINB, G><<<blocks, 256>>>(out, 4);
  cudaDeviceSynchronize();
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, probe_lds_g<BAR, MINB, G>);
  int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, probe_lds_g<BAR, MINB, G>, 256, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe_lds_g<BAR, MINB, G><<<blocks, 256>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double relax = (double)blocks * 256 * iters * 64 * 32;
  printf("{\"probe\": \"%s\", \"bar\": %d, \"minb\": %d, \"regs\": %d, \"spill\": %d, \"occ\": %d, \"ms\": %.3f, \"relax_per_clk_sm_at_max\": %.2f, \"err\": \"%s\"}\n",
         tag, BAR, MINB, fa.numRegs, (int)fa.localSizeBytes, occ, ms, relax / (ms * 1e-3) / (sms * (double)clk * 1e3),
         cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

// ---- pair pattern (round 2, session 5): both operands of the FADD2 are k-pairs -------------------
// s = (a_ik, a_i,k+1) + (b_kj, b_k+1,j) (one FADD2, no broadcast), x_ij = min(x_ij, s.lo, s.hi)
// (one FMNMX3 whose two candidates are the halves of ONE register pair). Needs B with k
// contiguous (the transposed pivot strip). Same instruction count per relaxation as the
// production pattern; different register-operand shape.
__device__ __forceinline__ unsigned long long fadd2p(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
template <int RM, int MINB>
__global__ void __launch_bounds__(256, MINB) probe_pair(float *out, int iters, float seed) {
  constexpr int NA = RM * 8;
  float x[NA];
  unsigned long long a[RM], b[8];
#pragma unroll
  for (int i = 0; i < NA; ++i) x[i] = 1e30f;
#pragma unroll
  for (int i = 0; i < RM; ++i) { float p = seed * (threadIdx.x + i), q = p + 1.f; asm("mov.b64 %0, {%1,%2};" : "=l"(a[i]) : "f"(p), "f"(q)); }
#pragma unroll
  for (int i = 0; i < 8; ++i) { float p = seed + i, q = seed - i; asm("mov.b64 %0, {%1,%2};" : "=l"(b[i]) : "f"(p), "f"(q)); }
  unsigned long long zero;
  { float z0 = 0.f; asm("mov.b64 %0, {%1,%1};" : "=l"(zero) : "f"(z0)); }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(b[i]) : "l"(zero));
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      unsigned long long s[RM];
#pragma unroll
      for (int r = 0; r < RM; ++r) s[r] = fadd2p(a[r], b[c]);
#pragma unroll
      for (int r = 0; r < RM; ++r) min3v(x[8 * r + c], lo(s[r]), hi(s[r]));
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NA; ++i) s += x[i];
  if (s == 1.2345f) out[threadIdx.x] = s;
}
template <int RM, int MINB>
void run_pair(const char *tag, float *out, int sms, int clk) {
  const int iters = 4000;
  const int blocks = sms * MINB * 8;
  probe_pair<RM, MINB><<<blocks, 256>>>(out, 10, 1.0001f);
  cudaDeviceSynchronize();
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, probe_pair<RM, MINB>);
  int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, probe_pair<RM, MINB>, 256, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe_pair<RM, MINB><<<blocks, 256>>>(out, iters, 1.0001f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double relax = (double)blocks * 256 * iters * RM * 8 * 2;
  printf("{\"probe\": \"%s\", \"RM\": %d, \"minb\": %d, \"regs\": %d, \"spill\": %d, \"occ\": %d, \"ms\": %.3f, \"relax_per_clk_sm_at_max\": %.2f, \"err\": \"%s\"}\n",
         tag, RM, MINB, fa.numRegs, (int)fa.localSizeBytes, occ, ms, relax / (ms * 1e-3) / (sms * (double)clk * 1e3),
         cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

// The pair pattern fed from shared memory: A [i][k] and Bt [j][k], both padded to 36 floats per
// row (conflict-free LDS.128); thread (tx, ty) owns rows ty + 16 r and columns tx + 16 c. Per q
// (4 k): 8 LDS.128 of A (held), then per column one LDS.128 of Bt and 16 FADD2 + 16 FMNMX3.
template <int BAR, int MINB>
__global__ void __launch_bounds__(256, MINB) probe_lds_pair(float *out, int iters) {
  constexpr int AS = 36;
  __shared__ __align__(16) float as_[128 * AS + 4];
  __shared__ __align__(16) float bs_[128 * AS + 4];
  for (int e = threadIdx.x; e < 128 * AS + 4; e += 256) { as_[e] = 1.0f + (e % 97); bs_[e] = 2.0f + (e % 89); }
  __syncthreads();
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 1e30f;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const int st = (it & 1) * 4;
    const float *as = as_ + ty * AS + st;
    const float *bs = bs_ + tx * AS + st;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 a[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) a[r] = *reinterpret_cast<const float4 *>(as + 16 * r * AS + 4 * q);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 b = *reinterpret_cast<const float4 *>(bs + 16 * c * AS + 4 * q);
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          float2 s[4], t[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) s[r] = __fadd2_rn(make_float2(a[4 * g + r].x, a[4 * g + r].y), make_float2(b.x, b.y));
#pragma unroll
          for (int r = 0; r < 4; ++r) t[r] = __fadd2_rn(make_float2(a[4 * g + r].z, a[4 * g + r].w), make_float2(b.z, b.w));
#pragma unroll
          for (int r = 0; r < 4; ++r) acc[4 * g + r][c] = fminf(acc[4 * g + r][c], fminf(s[r].x, s[r].y));
#pragma unroll
          for (int r = 0; r < 4; ++r) acc[4 * g + r][c] = fminf(acc[4 * g + r][c], fminf(t[r].x, t[r].y));
        }
      }
    }
    if (BAR) __syncthreads();
  }
  float s = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[r][c];
  if (s == 1.2345f) out[threadIdx.x] = s;
}
template <int BAR, int MINB>
void run_lds_pair(const char *tag, float *out, int sms, int clk) {
  const int iters = 400;
  const int blocks = sms * 2 * 8;
  probe_lds_pair<BAR, MINB><<<blocks, 256>>>(out, 4);
  cudaDeviceSynchronize();
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, probe_lds_pair<BAR, MINB>);
  int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, probe_lds_pair<BAR, MINB>, 256, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe_lds_pair<BAR, MINB><<<blocks, 256>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double relax = (double)blocks * 256 * iters * 64 * 32;
  printf("{\"probe\": \"%s\", \"bar\": %d, \"minb\": %d, \"regs\": %d, \"spill\": %d, \"occ\": %d, \"ms\": %.3f, \"relax_per_clk_sm_at_max\": %.2f, \"err\": \"%s\"}\n",
         tag, BAR, MINB, fa.numRegs, (int)fa.localSizeBytes, occ, ms, relax / (ms * 1e-3) / (sms * (double)clk * 1e3),
         cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *out; cudaMalloc(&out, 4096 * 4); cudaMemset(out, 0xff, 4096 * 4);
  run_lds<0, 2>("lds-nobar", out, sms, clk);
  run_lds<1, 2>("lds-bar-per-32k", out, sms, clk);
  run<8, 2, 0>("64acc-16w", out, sms, clk);
  run<8, 2, 1>("64acc-16w-inter", out, sms, clk);
  run<4, 4, 0>("32acc-32w", out, sms, clk);
  run<4, 4, 1>("32acc-32w-inter", out, sms, clk);
  run<4, 2, 0>("32acc-16w", out, sms, clk);
  run<8, 1, 0>("64acc-8w", out, sms, clk);
  run<2, 4, 0>("16acc-32w", out, sms, clk);
  run<8, 2, 0>("64acc-16w-again", out, sms, clk);
  run<8, 2, 3>("scalar-pairs-64acc-16w", out, sms, clk);
  run<8, 2, 5>("cross-prodFADD2-pairFMNMX3-64acc-16w", out, sms, clk);
  run<8, 2, 6>("boustrophedon-64acc-16w", out, sms, clk);
  run<8, 2, 64 + 4>("bbfence-G4", out, sms, clk);
  run<8, 2, 64 + 8>("bbfence-G8", out, sms, clk);
  run<8, 2, 16 + 4>("fence-warpsync-G4", out, sms, clk);
  run<8, 2, 16 + 8>("fence-warpsync-G8", out, sms, clk);
  run<8, 2, 32 + 4>("fence-1warpsync-G4", out, sms, clk);
  run<8, 2, 32 + 8>("fence-1warpsync-G8", out, sms, clk);
  run_lds_g<1, 2, 1>("lds-G1", out, sms, clk);
  run_lds_g<1, 2, 2>("lds-G2", out, sms, clk);
  run_lds_g<1, 2, 4>("lds-G4", out, sms, clk);
  run<8, 2, 2>("breuse-G2-64acc-16w", out, sms, clk);
  run<8, 2, 4>("breuse-G4-64acc-16w", out, sms, clk);
  run<8, 2, 8>("breuse-G8-64acc-16w", out, sms, clk);
  run<8, 1, 8>("breuse-G8-64acc-8w", out, sms, clk);
  run_pair<8, 2>("pair-64acc-16w", out, sms, clk);
  run_pair<4, 4>("pair-32acc-32w", out, sms, clk);
  run_pair<4, 2>("pair-32acc-16w", out, sms, clk);
  run_pair<8, 1>("pair-64acc-8w", out, sms, clk);
  run_lds_pair<0, 2>("pair-lds-nobar", out, sms, clk);
  run_lds_pair<1, 2>("pair-lds-bar-per-32k", out, sms, clk);
  return 0;
}

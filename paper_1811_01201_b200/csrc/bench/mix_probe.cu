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
  for (int it = 0; it < iters; ++it) {
    // loop-carried B operands (b + 0, not foldable because of signed zero): without this
    // ptxas CSEs the FADD2s across iterations (8 extra FADD2 per 8*RM, not counted)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(b[i]) : "l"(zero));
#pragma unroll
    for (int r = 0; r < RM; ++r) {
      if (ORDER == 0) {   // production order: per 4 columns: 4 FADD2 then 4 FMNMX3
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

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *out; cudaMalloc(&out, 4096 * 4);
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
  return 0;
}

// Microkernel probe (development tool): the phase-3 8x8 register-blocked FADD2+FMNMX3
// inner loop fed from shared memory, with no global loads and no barriers in the loop.
// Separates the instruction-mix limit from the staging / synchronisation overheads.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

template <int MODE>
__global__ void __launch_bounds__(256, 2) mk(float *out, int iters) {
  constexpr int TN = 128, AS = 36;
  __shared__ __align__(16) float as_[128 * AS];
  __shared__ __align__(16) float bs_[32 * TN];
  for (int e = threadIdx.x; e < 128 * AS; e += 256) as_[e] = 1.0f + (e % 97);
  for (int e = threadIdx.x; e < 32 * TN; e += 256) bs_[e] = 2.0f + (e % 89);
  __syncthreads();
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const float *as = as_ + ty * AS;
  const float *bs = bs_ + tx * 4;
  float acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 1e30f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 b[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) b[c] = *reinterpret_cast<const float4 *>(bs + (q * TN + 16 * c) * 4);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const float4 a = *reinterpret_cast<const float4 *>(as + 16 * r * AS + 4 * q);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (MODE == 0) {
            const float2 s01 = __fadd2_rn(make_float2(a.x, a.y), make_float2(b[c].x, b[c].y));
            const float2 s23 = __fadd2_rn(make_float2(a.z, a.w), make_float2(b[c].z, b[c].w));
            acc[r][c] = fminf(acc[r][c], fminf(s01.x, s01.y));
            acc[r][c] = fminf(acc[r][c], fminf(s23.x, s23.y));
          } else if (MODE == 1) {   // scalar FADD + FMNMX3
            acc[r][c] = fminf(acc[r][c], fminf(a.x + b[c].x, a.y + b[c].y));
            acc[r][c] = fminf(acc[r][c], fminf(a.z + b[c].z, a.w + b[c].w));
          } else if (MODE == 2) {   // integer VIADDMNMX on the same data bits
            int x = __float_as_int(acc[r][c]);
            x = __viaddmin_s32(__float_as_int(a.x), __float_as_int(b[c].x), x);
            x = __viaddmin_s32(__float_as_int(a.y), __float_as_int(b[c].y), x);
            x = __viaddmin_s32(__float_as_int(a.z), __float_as_int(b[c].z), x);
            x = __viaddmin_s32(__float_as_int(a.w), __float_as_int(b[c].w), x);
            acc[r][c] = __int_as_float(x);
          } else if (MODE == 3) {   // half FADD2 pairs, half scalar FADD (pipe balance)
            const float2 s01 = __fadd2_rn(make_float2(a.x, a.y), make_float2(b[c].x, b[c].y));
            acc[r][c] = fminf(acc[r][c], fminf(s01.x, s01.y));
            acc[r][c] = fminf(acc[r][c], fminf(a.z + b[c].z, a.w + b[c].w));
          }
        }
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[r][c];
  if (s == 12345.f) out[threadIdx.x] = s;
}

template <int MODE>
void run(float *out, int sms, int clk, int blocks_per_sm) {
  const int iters = 200;
  dim3 g(sms * blocks_per_sm * 4);
  mk<MODE><<<g, 256>>>(out, iters);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mk<MODE><<<g, 256>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double relax = (double)g.x * 256 * 64 * 32 * iters;
  printf("{\"mode\": %d, \"ms\": %.3f, \"relax_per_clk_sm_at_max\": %.2f, \"err\": \"%s\"}\n", MODE, ms,
         relax / (ms * 1e-3) / (sms * (double)clk * 1e3), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *out; cudaMalloc(&out, 4096 * 4);
  run<0>(out, sms, clk, 2); run<1>(out, sms, clk, 2); run<2>(out, sms, clk, 2); run<3>(out, sms, clk, 2);
  run<0>(out, sms, clk, 2);
  return 0;
}

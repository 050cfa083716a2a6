// Pipe-mix probe (development tool): can the integer fused add+min (VIADDMNMX) run beside the
// FP32 FADD2 + FMNMX3 relaxation pair on other pipes, so that a tile splitting its columns
// between the two forms relaxes more per clock than either alone? One CTA of 1024 threads per
// SM, CH independent chains per thread; prints relaxations per clock per SM for each mix.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;
constexpr int CH = 8;

__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long x; asm("mov.b64 %0, {%1,%2};" : "=l"(x) : "f"(a), "f"(b)); return x;
}

// NF FADD2+FMNMX3 pairs (2 relaxations each, FP chains) and NI VIADDMNMX (1 relaxation each,
// integer chains) per chain step
template <int NF, int NI>
__global__ void __launch_bounds__(1024) mix(float *sink, long long *cyc, float seed) {
  float a[CH], b[CH], acc[CH];
  int ia[CH], ib[CH], iacc[CH];
  for (int c = 0; c < CH; ++c) {
    a[c] = seed * (threadIdx.x + c); b[c] = seed + c; acc[c] = 1e30f;
    ia[c] = threadIdx.x + c; ib[c] = c * 3; iacc[c] = 1 << 29;
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        unsigned long long x = pk(a[c], b[c]), y = pk(seed, seed);
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(y));
        asm("mov.b64 {%0,%1}, %2;" : "=f"(a[c]), "=f"(b[c]) : "l"(x));
        asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(acc[c]) : "f"(a[c]), "f"(b[c]));
      }
#pragma unroll
      for (int i = 0; i < NI; ++i) iacc[c] = __viaddmin_s32(iacc[c], ib[c], ia[c] + i);
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c] + a[c] + b[c] + (float)iacc[c];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int NF, int NI>
int run(int sms) {
  float *sink; long long *cyc;
  cudaMalloc(&sink, sizeof(float) * sms * 1024);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  mix<NF, NI><<<sms, 1024>>>(sink, cyc, 1.0001f);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mix<NF, NI><<<sms, 1024>>>(sink, cyc, 1.0001f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  long long h[1024]; cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double mean = 0; for (int i = 0; i < sms; ++i) mean += h[i]; mean /= sms;
  const double relax = (double)ITERS * CH * (2.0 * NF + NI) * 1024;   // per CTA = per SM
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"NF\": %d, \"NI\": %d, \"relax_per_clk_per_sm\": %.2f, \"ms\": %.4f, \"err\": \"%s\"}\n", NF, NI,
         relax / mean, ms, cudaGetErrorString(cudaGetLastError()));
  cudaFree(sink); cudaFree(cyc);
  return 0;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<1, 0>(sms); run<0, 1>(sms); run<0, 2>(sms); run<1, 1>(sms); run<2, 1>(sms); run<1, 2>(sms);
  run<3, 1>(sms); run<4, 1>(sms); run<2, 2>(sms);
  return 0;
}

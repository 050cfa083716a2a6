// Explorer (development tool): the library's phase-3 tile kernel with a 256-deep k range (two
// rounds in one pass, one epilogue) against two 128-deep launches, on the same n = 16384
// key-encoded data: relaxations / clock / SM of each ("two rounds per pass").
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <vector>
#include "../fw_kernels.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

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
      init[i * n + j] = (float)(w * 128 + (j & 127));
    }
  float *D; int32_t *P; int *mk;
  CK(cudaMalloc(&D, n * n * 4)); CK(cudaMalloc(&P, n * n * 4)); CK(cudaMalloc(&mk, 4));
  auto lib = fwb::minplus_tile_kernel<float, 128, 128, fwb::MODE_KEY, false>;
  const int lbytes = fwb::TileShape<128, 128>::kBytes;
  CK(cudaFuncSetAttribute(lib, cudaFuncAttributeMaxDynamicSharedMemorySize, lbytes));
  const int kb = 128 * 50;
  dim3 g(n / 128, n / 128);
  auto args = [&](int k0, int kd) {
    fwb::TileArgs a{};
    a.ld = n; a.B = D + (int64_t)k0 * n; a.ldb = n; a.kb = k0; a.Kd = kd;
    a.rows_lim = (int)n; a.cols_lim = (int)n;
    a.mr_lo[0] = kb; a.mr_hi[0] = kb + 512; a.mc_lo[0] = kb; a.mc_hi[0] = kb + 512;   // both blocks' strips
    return a;
  };
  const fwb::TileArgs a1 = args(kb, 128), a2 = args(kb + 128, 128), a12 = args(kb, 256), a14 = args(kb, 512);
  const int64_t tiles = (n / 128 - 4) * (n / 128 - 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int pass = 0; pass < 2; ++pass)
    for (int which = 0; which < 3; ++which) {
      CK(cudaMemcpy(D, init.data(), n * n * 4, cudaMemcpyHostToDevice));
      auto launch = [&]() {
        if (which == 0) { lib<<<g, 256, lbytes>>>(D, P, a1, mk); lib<<<g, 256, lbytes>>>(D, P, a2, mk); }
        else if (which == 1) lib<<<g, 256, lbytes>>>(D, P, a12, mk);
        else lib<<<g, 256, lbytes>>>(D, P, a14, mk);
      };
      launch(); launch();
      CK(cudaDeviceSynchronize());
      const int reps = 10;
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
      const double relax = (double)tiles * 128 * 128 * (which == 2 ? 512 : 256);
      printf("{\"variant\": \"%s\", \"ms\": %.4f, \"relax_per_clk_sm_at_max_clock\": %.2f}\n",
             which == 0 ? "two 128-deep launches" : which == 1 ? "one 256-deep launch" : "one 512-deep launch", ms,
             relax / (ms * 1e-3) / (sms * (double)clk * 1e3));
      fflush(stdout);
    }
  return 0;
}

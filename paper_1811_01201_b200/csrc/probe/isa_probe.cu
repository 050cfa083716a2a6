// L0 ISA / clock probe for the min-plus relaxation on sm_100a.
// Measures sustained per-SM throughput of the instructions a relaxation
// d = min(d, a + b) can compile to: FADD, FADD2 (add.rn.f32x2), FMNMX, FMNMX3
// (3-input min.f32), VIADDMNMX (__viaddmin_s32), VIMNMX3, IADD, and the
// per-relaxation select chain (FADD+FSETP+FSEL+SEL) that a naive P update needs.
// One CTA of 1024 threads per SM, 148+ CTAs; each CTA times itself with clock64.
// Prints one JSON object per probe: ops (lane-ops) per clock per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 2048;
constexpr int CH = 8;  // independent chains per thread

__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long x; asm("mov.b64 %0, {%1,%2};" : "=l"(x) : "f"(a), "f"(b)); return x;
}

// op ids
enum { OP_FADD, OP_FADD2, OP_FMNMX, OP_FMNMX3, OP_MIX_FADD2_FMNMX3, OP_VIADDMNMX,
       OP_VIMNMX3, OP_IADD_VIMNMX3, OP_SELECT, OP_FADD_FMNMX,
       OP_MIX_PINGPONG, OP_MIX_OWN_SCALAR, OP_MIX_PAIR_PAIR, OP_MIX_BCAST_FIRST, OP_COUNT };
static const char* NAMES[] = {"FADD", "FADD2", "FMNMX", "FMNMX3", "FADD2+FMNMX3",
  "VIADDMNMX", "VIMNMX3", "IADD+VIMNMX3", "FADD+FSETP+FSEL+SEL", "FADD+FMNMX",
  "mix: FADD2 not in place (x2 = x + y, x = x2 + y)", "mix: own scalar per chain", "mix: pair + pair in place",
  "mix: scalar + pair -> fresh pair (production form), FMNMX3 on its halves"};
// relaxation-equivalents (lane-ops counted as relaxations) per inner step per chain
static const double RELAX_PER_STEP[] = {1, 2, 2, 2, 2, 1, 3, 2, 1, 1, 4, 2, 2, 2};  // lane-ops per step

template <int OP>
__global__ void __launch_bounds__(1024) probe(float* sink, long long* cyc, float seed) {
  float a[CH], b[CH], acc[CH];
  int ia[CH], ib[CH], iacc[CH];
  int q[CH];
  for (int c = 0; c < CH; ++c) {
    a[c] = seed * (threadIdx.x + c); b[c] = seed + c; acc[c] = 1e30f;
    ia[c] = threadIdx.x + c; ib[c] = c * 3; iacc[c] = 1 << 29; q[c] = 0;
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == OP_FADD) {
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(acc[c]) : "f"(b[c]));
      } else if (OP == OP_FADD2) {
        unsigned long long x = pk(acc[c], a[c]), y = pk(b[c], b[c]);
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(y));
        asm("mov.b64 {%0,%1}, %2;" : "=f"(acc[c]), "=f"(a[c]) : "l"(x));
      } else if (OP == OP_FMNMX) {
        // acc chain with a loop-carried second operand so ptxas cannot fuse into FMNMX3
        asm volatile("min.f32 %0, %0, %1;" : "+f"(acc[c]) : "f"(a[c]));
        asm volatile("max.f32 %0, %0, %1;" : "+f"(a[c]) : "f"(acc[c]));
      } else if (OP == OP_FMNMX3) {
        asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(acc[c]) : "f"(b[c]), "f"(a[c]));
      } else if (OP == OP_MIX_FADD2_FMNMX3) {
        // x <- x + y (packed, loop-carried), acc <- min(acc, x.lo, x.hi)
        unsigned long long x = pk(a[c], b[c]), y = pk(seed, seed);
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(y));
        asm("mov.b64 {%0,%1}, %2;" : "=f"(a[c]), "=f"(b[c]) : "l"(x));
        asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(acc[c]) : "f"(a[c]), "f"(b[c]));
      } else if (OP == OP_MIX_PINGPONG) {
        // two steps: x2 = x + y, acc = min(acc, x2); x = x2 + y, acc = min(acc, x) — destinations differ from sources
        unsigned long long x = pk(a[c], b[c]), y = pk(seed, seed), x2;
        asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(x2) : "l"(x), "l"(y));
        float p, q; asm("mov.b64 {%0,%1}, %2;" : "=f"(p), "=f"(q) : "l"(x2));
        asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(acc[c]) : "f"(p), "f"(q));
        asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(x) : "l"(x2), "l"(y));
        asm("mov.b64 {%0,%1}, %2;" : "=f"(a[c]), "=f"(b[c]) : "l"(x));
        asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(acc[c]) : "f"(a[c]), "f"(b[c]));
      } else if (OP == OP_MIX_OWN_SCALAR) {
        // every chain adds its own broadcast scalar (nothing shared between consecutive FADD2s)
        float sc = __int_as_float(ia[c]);
        unsigned long long x = pk(a[c], b[c]), y = pk(sc, sc);
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(y));
        asm("mov.b64 {%0,%1}, %2;" : "=f"(a[c]), "=f"(b[c]) : "l"(x));
        asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(acc[c]) : "f"(a[c]), "f"(b[c]));
      } else if (OP == OP_MIX_PAIR_PAIR) {
        // every chain adds its own PAIR (two registers): the pair + pair form, in place
        unsigned long long x = pk(a[c], b[c]), y = pk(__int_as_float(ia[c]), __int_as_float(ib[c]));
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(y));
        asm("mov.b64 {%0,%1}, %2;" : "=f"(a[c]), "=f"(b[c]) : "l"(x));
        asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(acc[c]) : "f"(a[c]), "f"(b[c]));
      } else if (OP == OP_MIX_BCAST_FIRST) {
        // production form: fresh result pair = own scalar (broadcast) + a loop-invariant pair; FMNMX3 on its halves;
        // the scalar is loop-carried through the accumulator's chain so nothing is hoisted
        float sc = acc[c];
        unsigned long long y = pk(a[c], b[c]), s2, t = pk(sc, sc);
        asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(s2) : "l"(t), "l"(y));
        float p, q; asm("mov.b64 {%0,%1}, %2;" : "=f"(p), "=f"(q) : "l"(s2));
        asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(acc[c]) : "f"(p), "f"(q));
      } else if (OP == OP_VIADDMNMX) {
        iacc[c] = __viaddmin_s32(iacc[c], ib[c], ia[c]);   // min(iacc+ib, ia): loop-carried
      } else if (OP == OP_VIMNMX3) {
        asm volatile("min.s32 %0, %0, %1;" : "+r"(iacc[c]) : "r"(ia[c]));
        asm volatile("min.s32 %0, %0, %1;" : "+r"(iacc[c]) : "r"(ib[c]));
        asm volatile("max.s32 %0, %0, %1;" : "+r"(ia[c]) : "r"(iacc[c]));
      } else if (OP == OP_IADD_VIMNMX3) {
        asm volatile("add.s32 %0, %0, %1;" : "+r"(ia[c]) : "r"(ib[c]));
        asm volatile("add.s32 %0, %0, %1;" : "+r"(q[c]) : "r"(ib[c]));
        iacc[c] = min(iacc[c], min(ia[c], q[c]));
      } else if (OP == OP_SELECT) {
        float s; asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(s) : "f"(a[c]), "f"(b[c]));
        bool lt = s < acc[c];
        acc[c] = lt ? s : acc[c];
        q[c] = lt ? it : q[c];
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[c]) : "f"(seed));
      } else if (OP == OP_FADD_FMNMX) {
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[c]) : "f"(b[c]));
        asm volatile("min.f32 %0, %0, %1;" : "+f"(acc[c]) : "f"(a[c]));
      }
    }
  }
  long long t1 = clock64();
  float r = 0.f; int ir = 0;
  for (int c = 0; c < CH; ++c) { r += acc[c] + a[c]; ir += iacc[c] + q[c] + ia[c]; }
  if (r == 1234.5f && ir == 77) sink[threadIdx.x] = r;  // keep everything live
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
static int run(int sms, float* sink, long long* dcyc, long long* hcyc) {
  const int blocks = sms, threads = 1024;
  probe<OP><<<blocks, threads>>>(sink, dcyc, 1.0001f);  // warm-up
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<OP><<<blocks, threads>>>(sink, dcyc, 1.0001f);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  CK(cudaMemcpy(hcyc, dcyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost));
  long long mx = 0; double mean = 0;
  for (int i = 0; i < blocks; ++i) { mx = hcyc[i] > mx ? hcyc[i] : mx; mean += hcyc[i]; }
  mean /= blocks;
  double ops_per_block = (double)threads * ITERS * CH * RELAX_PER_STEP[OP];
  double per_clk_sm = ops_per_block / mean;
  double mhz = mean / (ms * 1e3);
  printf("{\"probe\": \"%s\", \"relax_per_clk_per_sm\": %.2f, \"cycles_mean\": %.0f, \"cycles_max\": %lld, "
         "\"ms\": %.4f, \"eff_mhz\": %.0f, \"relax_per_s_chip\": %.4e}\n",
         NAMES[OP], per_clk_sm, mean, mx, ms, mhz, per_clk_sm * sms * mhz * 1e6);
  return 0;
}

int main() {
  int dev = 0, sms = 0, clk = 0, smem = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  CK(cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
  printf("{\"sms\": %d, \"clock_rate_khz\": %d, \"smem_per_sm\": %d}\n", sms, clk, smem);
  float* sink; long long* dcyc; long long* hcyc = new long long[sms];
  CK(cudaMalloc(&sink, 4096 * sizeof(float)));
  CK(cudaMalloc(&dcyc, sms * sizeof(long long)));
  int rc = 0;
  rc |= run<OP_FADD>(sms, sink, dcyc, hcyc);
  rc |= run<OP_FADD2>(sms, sink, dcyc, hcyc);
  rc |= run<OP_FMNMX>(sms, sink, dcyc, hcyc);
  rc |= run<OP_FMNMX3>(sms, sink, dcyc, hcyc);
  rc |= run<OP_MIX_FADD2_FMNMX3>(sms, sink, dcyc, hcyc);
  rc |= run<OP_FADD_FMNMX>(sms, sink, dcyc, hcyc);
  rc |= run<OP_VIADDMNMX>(sms, sink, dcyc, hcyc);
  rc |= run<OP_VIMNMX3>(sms, sink, dcyc, hcyc);
  rc |= run<OP_IADD_VIMNMX3>(sms, sink, dcyc, hcyc);
  rc |= run<OP_SELECT>(sms, sink, dcyc, hcyc);
  rc |= run<OP_MIX_PINGPONG>(sms, sink, dcyc, hcyc);
  rc |= run<OP_MIX_OWN_SCALAR>(sms, sink, dcyc, hcyc);
  rc |= run<OP_MIX_PAIR_PAIR>(sms, sink, dcyc, hcyc);
  rc |= run<OP_MIX_BCAST_FIRST>(sms, sink, dcyc, hcyc);
  return rc;
}

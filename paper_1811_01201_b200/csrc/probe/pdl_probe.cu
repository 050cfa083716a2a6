// Programmatic dependent launch probe (development only): does a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization start its CTAs before the previous kernel
// in the stream has finished, when event records / waits sit between the two launches?
// Kernel A: 2 CTAs per SM, CTA b spins (1 + b % 8) * 20 us, triggers its dependents at start.
// Kernel B: each CTA stamps its start, griddepcontrol.wait, stamps again.
// Prints A's last end, B's first start and B's first post-wait stamp (ns, globaltimer).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void kA(unsigned long long *aend) {
  asm volatile("griddepcontrol.launch_dependents;");
  const uint64_t t0 = gtime(), dur = (1 + blockIdx.x % 8) * 20000ull;
  while (gtime() - t0 < dur) {
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(aend, (unsigned long long)gtime());
}

__global__ void kB(unsigned long long *bstart, unsigned long long *bwait) {
  const uint64_t t = gtime();
  if (threadIdx.x == 0) atomicMin(bstart, (unsigned long long)t);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) atomicMin(bwait, (unsigned long long)gtime());
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *d;
  cudaMalloc(&d, 3 * sizeof(unsigned long long));
  cudaStream_t st, side;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
  cudaEvent_t e0, e1, e2;
  cudaEventCreateWithFlags(&e0, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&e1, cudaEventDisableTiming);
  cudaEventCreate(&e2);
  const char *names[4] = {"adjacent", "event record between", "wait on a done event between",
                          "record + wait + timing record between"};
  for (int variant = 0; variant < 4; ++variant)
    for (int rep = 0; rep < 2; ++rep) {
      unsigned long long init[3] = {0ull, ~0ull, ~0ull};
      cudaMemcpy(d, init, sizeof init, cudaMemcpyHostToDevice);
      cudaEventRecord(e0, side);   // completes immediately
      cudaDeviceSynchronize();
      kA<<<2 * sms * 4, 256, 0, st>>>(d);
      if (variant == 1 || variant == 3) cudaEventRecord(e1, st);
      if (variant == 2 || variant == 3) cudaStreamWaitEvent(st, e0, 0);
      if (variant == 3) cudaEventRecord(e2, st);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(2 * sms);
      cfg.blockDim = dim3(256);
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaError_t err = cudaLaunchKernelEx(&cfg, kB, d + 1, d + 2);
      cudaDeviceSynchronize();
      unsigned long long h[3];
      cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      printf("{\"variant\": \"%s\", \"rep\": %d, \"launch\": \"%s\", \"b_start_minus_a_end_us\": %.2f, "
             "\"b_wait_minus_a_end_us\": %.2f}\n",
             names[variant], rep, cudaGetErrorString(err), ((double)h[1] - (double)h[0]) / 1e3,
             ((double)h[2] - (double)h[0]) / 1e3);
    }
  return 0;
}

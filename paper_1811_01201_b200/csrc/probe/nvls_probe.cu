// NVLS (switch multicast) feasibility probe on one GPU (development tool): multicast object
// with one device, fabric-handle export, physical memory bind, unicast + multicast mappings,
// multimem.st of v4.f32 data and a release-ordered u64 flag, read back through the unicast
// mapping. Prints one line per step.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#define CK(x) do { CUresult r = (x); const char *s = nullptr; cuGetErrorString(r, &s); \
  printf("%-60s -> %d %s\n", #x, (int)r, s ? s : ""); if (r != CUDA_SUCCESS) return 1; } while (0)

__global__ void pub(float *mc, unsigned long long *mcflag, int n, unsigned long long tag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (4 * i < n) {
    float a = 4 * i, b = 4 * i + 1, c = 4 * i + 2, d = 4 * i + 3;
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + 4 * i), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" ::"l"(mcflag), "l"(tag) : "memory");
  }
}
__global__ void waitk(const unsigned long long *flag, unsigned long long want, int *ok) {
  unsigned long long v = 0;
  for (int it = 0; it < 1000000; ++it) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= want) break;
    __nanosleep(100);
  }
  *ok = (v >= want);
}

int main() {
  CK(cuInit(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
  int mcs = 0; cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  printf("multicast supported: %d\n", mcs);
  CUmulticastObjectProp mp; memset(&mp, 0, sizeof mp);
  mp.numDevices = 1; mp.size = 1 << 21; mp.handleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
  size_t gmin = 0, grec = 0;
  CK(cuMulticastGetGranularity(&gmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  CK(cuMulticastGetGranularity(&grec, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  printf("granularity min %zu rec %zu\n", gmin, grec);
  size_t size = ((size_t)(8 << 20) + grec - 1) / grec * grec;
  mp.size = size;
  CUmemGenericAllocationHandle mc;
  CUresult cr = CUDA_ERROR_UNKNOWN;
  const CUmemAllocationHandleType hts[3] = {CU_MEM_HANDLE_TYPE_FABRIC, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_NONE};
  for (int nd = 1; nd <= 2 && cr != CUDA_SUCCESS; ++nd)
    for (int h = 0; h < 3 && cr != CUDA_SUCCESS; ++h) {
      mp.numDevices = nd; mp.handleTypes = hts[h];
      cr = cuMulticastCreate(&mc, &mp);
      printf("cuMulticastCreate(numDevices=%d, handleTypes=%d) -> %d\n", nd, (int)hts[h], (int)cr);
    }
  if (cr != CUDA_SUCCESS) return 1;
  CUmemFabricHandle fh;
  cr = cuMemExportToShareableHandle(&fh, mc, CU_MEM_HANDLE_TYPE_FABRIC, 0);
  printf("export fabric handle -> %d\n", (int)cr);
  CK(cuMulticastAddDevice(mc, dev));
  CUmemAllocationProp ap; memset(&ap, 0, sizeof ap);
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = dev;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
  size_t ag = 0; CK(cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  printf("alloc granularity %zu\n", ag);
  CUmemGenericAllocationHandle ph;
  cr = cuMemCreate(&ph, size, &ap, 0);
  printf("cuMemCreate(FABRIC) -> %d\n", (int)cr);
  if (cr != CUDA_SUCCESS) { ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_NONE; CK(cuMemCreate(&ph, size, &ap, 0)); }
  CK(cuMulticastBindMem(mc, 0, ph, 0, size, 0));
  CUdeviceptr uc, mcp;
  CK(cuMemAddressReserve(&uc, size, 0, 0, 0)); CK(cuMemMap(uc, size, 0, ph, 0));
  CK(cuMemAddressReserve(&mcp, size, 0, 0, 0)); CK(cuMemMap(mcp, size, 0, mc, 0));
  CUmemAccessDesc ad; ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = dev; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, size, &ad, 1)); CK(cuMemSetAccess(mcp, size, &ad, 1));
  CK(cuMemsetD8(uc, 0, size));
  const int n = 1 << 20;
  unsigned long long *flag_uc = (unsigned long long *)(uc + size - 256), *flag_mc = (unsigned long long *)(mcp + size - 256);
  int *ok; cudaMalloc(&ok, 4);
  pub<<<n / 4 / 256, 256>>>((float *)mcp, flag_mc, n, 5);
  waitk<<<1, 1>>>(flag_uc, 5ull * (n / 4 / 256), ok);
  printf("kernels: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  float *h = new float[n]; int hok = 0;
  cudaMemcpy(h, (void *)uc, n * 4, cudaMemcpyDeviceToHost); cudaMemcpy(&hok, ok, 4, cudaMemcpyDeviceToHost);
  unsigned long long hf = 0; cudaMemcpy(&hf, flag_uc, 8, cudaMemcpyDeviceToHost);
  int bad = 0; for (int i = 0; i < n; ++i) bad += h[i] != (float)i;
  printf("multimem data bad=%d flag=%llu wait_ok=%d\n", bad, hf, hok);
  // bandwidth: multimem.st of 64 MiB-equivalent through the 8 MiB window
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 20; ++r) pub<<<n / 4 / 256, 256>>>((float *)mcp, flag_mc, n, 1);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("multimem.st %.1f GB/s (1 device)\n", 20.0 * n * 4 / (ms * 1e-3) / 1e9);
  return 0;
}

// Reuse-cache experiment (development probe): the production operand pattern
// (FADD2 broadcast scalar + pair, FMNMX3 on two pairs) in the row-group order ptxas turns into
// b0 b1 b0 b1 ... ; compiled to a cubin whose .reuse control bits tools/reuse_patch.py edits.
// Results are written out so a patched run can be compared bit for bit with the original.
__device__ __forceinline__ unsigned long long fadd2b(float a, unsigned long long b) {
  unsigned long long r;
  asm volatile("{ .reg .b64 t; mov.b64 t, {%1, %1}; add.rn.f32x2 %0, t, %2; }" : "=l"(r) : "f"(a), "l"(b));
  return r;
}
__device__ __forceinline__ void min3v(float &x, float p, float q) {
  asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(x) : "f"(p), "f"(q));
}
__device__ __forceinline__ float lo(unsigned long long v) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return a; }
__device__ __forceinline__ float hi(unsigned long long v) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return b; }

template <int G>
__device__ __forceinline__ void body(float *out, const float *in, int iters) {
  constexpr int RM = 8, NA = 64;
  float x[NA], a[2 * RM];
  unsigned long long b[8];
#pragma unroll
  for (int i = 0; i < NA; ++i) x[i] = 1e30f;
#pragma unroll
  for (int i = 0; i < 2 * RM; ++i) a[i] = in[(threadIdx.x * 16 + i) & 4095];
#pragma unroll
  for (int i = 0; i < 8; ++i) { float p = in[(threadIdx.x * 7 + 2 * i) & 4095], q = in[(threadIdx.x * 5 + 2 * i + 1) & 4095]; asm("mov.b64 %0, {%1,%2};" : "=l"(b[i]) : "f"(p), "f"(q)); }
  unsigned long long inc;
  { float z0 = in[4095]; asm("mov.b64 %0, {%1,%1};" : "=l"(inc) : "f"(z0)); }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(b[i]) : "l"(inc));   // b changes every iteration
#pragma unroll
    for (int r = 0; r < RM; r += G)
#pragma unroll
      for (int p = 0; p < 4; ++p) {
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
  float s = 0;
#pragma unroll
  for (int i = 0; i < NA; ++i) s += x[i] * (float)(i + 1);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
extern "C" __global__ void __launch_bounds__(256, 2) reuse_g4(float *out, const float *in, int iters) { body<4>(out, in, iters); }
extern "C" __global__ void __launch_bounds__(256, 2) reuse_g8(float *out, const float *in, int iters) { body<8>(out, in, iters); }

// The k-pair pattern: FADD2 (a_k, a_k+1) + (b_k, b_k+1), FMNMX3 on the two halves of its result
// (one FADD2 per FMNMX3, so ptxas keeps the source order: 8 consecutive FADD2s share one pair).
extern "C" __global__ void __launch_bounds__(256, 2) reuse_pair(float *out, const float *in, int iters) {
  constexpr int RM = 8, NA = 64;
  float x[NA];
  unsigned long long a[RM], b[8];
#pragma unroll
  for (int i = 0; i < NA; ++i) x[i] = 1e30f;
#pragma unroll
  for (int i = 0; i < RM; ++i) { float p = in[(threadIdx.x * 16 + 2 * i) & 4095], q = in[(threadIdx.x * 16 + 2 * i + 1) & 4095]; asm("mov.b64 %0, {%1,%2};" : "=l"(a[i]) : "f"(p), "f"(q)); }
#pragma unroll
  for (int i = 0; i < 8; ++i) { float p = in[(threadIdx.x * 7 + 2 * i) & 4095], q = in[(threadIdx.x * 5 + 2 * i + 1) & 4095]; asm("mov.b64 %0, {%1,%2};" : "=l"(b[i]) : "f"(p), "f"(q)); }
  unsigned long long inc;
  { float z0 = in[4095]; asm("mov.b64 %0, {%1,%1};" : "=l"(inc) : "f"(z0)); }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(b[i]) : "l"(inc));
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      unsigned long long s[RM];
#pragma unroll
      for (int r = 0; r < RM; ++r) asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(s[r]) : "l"(a[r]), "l"(b[c]));
#pragma unroll
      for (int r = 0; r < RM; ++r) min3v(x[8 * r + c], lo(s[r]), hi(s[r]));
    }
  }
  float sum = 0;
#pragma unroll
  for (int i = 0; i < NA; ++i) sum += x[i] * (float)(i + 1);
  out[blockIdx.x * blockDim.x + threadIdx.x] = sum;
}

// The L0 mix probe's pattern (isa_probe.cu OP_MIX_FADD2_FMNMX3): x += y (packed, in place, y one
// broadcast scalar shared by every chain), acc = min(acc, x.lo, x.hi); 8 chains per thread.
// ptxas flags y's .reuse on every FADD2; `reuse_patch.py --clear` removes the flags.
extern "C" __global__ void __launch_bounds__(256) reuse_l0(float *out, const float *in, int iters) {
  constexpr int CH = 8;
  unsigned long long x[CH];
  float acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    float p = in[(threadIdx.x * 8 + c) & 4095], q = in[(threadIdx.x * 3 + c + 100) & 4095];
    asm("mov.b64 %0, {%1,%2};" : "=l"(x[c]) : "f"(p), "f"(q));
    acc[c] = 1e30f;
  }
  unsigned long long y;
  { float z0 = in[4095]; asm("mov.b64 %0, {%1,%1};" : "=l"(y) : "f"(z0)); }
  for (int it = 0; it < iters * 16; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x[c]) : "l"(y));
      min3v(acc[c], lo(x[c]), hi(x[c]));
    }
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c] * (float)(c + 1);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// FFMA vs FFMA2 (fma.rn.f32x2) issue throughput on sm_100a (dev microbenchmark).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t pk(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void fma2(uint64_t& d, uint64_t a, uint64_t b) { asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b)); }
template <int MODE>
__global__ void k(float* out, float s, int iters) {
  float a = threadIdx.x * 1e-3f, b = s + threadIdx.x * 1e-7f;
  if (MODE == 0) {
    float acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fmaf(acc[i], a, b);
    float r = 0; for (int i = 0; i < 16; ++i) r += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  } else {
    uint64_t acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = pk(i, i + 0.5f);
    const uint64_t A = pk(a, a + 1.f), B = pk(b, b * 0.5f);
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) { asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[i]) : "l"(A), "l"(B)); }
    float r = 0; for (int i = 0; i < 8; ++i) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(acc[i])); r += x + y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  }
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
  int dev; cudaGetDevice(&dev); int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 20000;
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<148 * 4, 512>>>(o, 1.0001f, iters); else k<1><<<148 * 4, 512>>>(o, 1.0001f, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fmas = 148.0 * 4 * 512 * iters * 16;
      printf("mode %s: %.3f ms, %.1f TFLOP/s (FMA=2 flops)\n", mode ? "FFMA2" : "FFMA ", ms, fmas * 2 / ms / 1e9);
    }
  }
  return 0;
}

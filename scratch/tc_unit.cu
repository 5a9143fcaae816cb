// Standalone tcgen05 unit checks (dev only): TMEM st/ld round trip, one tf32 MMA.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cuda_bf16.h>
#include "../paper_2203_06233_b200/csrc/apply_tc.cuh"
using namespace stapk;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("ERR %s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); } } while (0)

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
      "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31]));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__global__ void k_roundtrip(float* out, uint32_t* taddr_out) {
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (tid == 0) *taddr_out = tmem;
  float v[32];
  for (int i = 0; i < 32; ++i) v[i] = tid * 100 + i;
  tmem_st32(tmem + ((uint32_t)(warp * 32) << 16), v);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  float r[32];
  tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), r);
  for (int i = 0; i < 32; ++i) out[tid * 32 + i] = r[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
}

// One MMA: M=128, N=32, K=8.  A[m][i] (MN-major, A layout as apply_tc), B[n][i] (K-major).
template <int MASK>
__global__ void k_mma(const float* A, const float* B, float* out) {
  __shared__ __align__(1024) unsigned char sa[4096];
  __shared__ __align__(1024) unsigned char sb[1024];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  for (int idx = tid; idx < 8 * 32; idx += 128) {  // A chunks (i, mc): m = 4mc..4mc+3
    const int i = idx / 32, mc = idx % 32;
    float* dst = reinterpret_cast<float*>(sa + mc * 128 + i * 16);
    for (int q = 0; q < 4; ++q) dst[q] = A[(4 * mc + q) * 8 + i];
  }
  for (int idx = tid; idx < 32 * 8; idx += 128) {
    const int nn = idx / 8, i = idx % 8;
    const int off = (nn >> 3) * 256 + ((i >> 2) & 1) * 128 + (nn & 7) * 16 + (i & 3) * 4;
    *reinterpret_cast<float*>(sb + off) = B[nn * 8 + i];
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (tid == 0) {
    const uint32_t idesc = umma_idesc_tf32(128, 32);
    const uint64_t ad = umma_desc(smem_u32(sa), 4096, 128), bd = umma_desc(smem_u32(sb), 128, 256);
    if (MASK) {
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n}\n" ::"r"(tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(0), "r"(0), "r"(0), "r"(0), "r"(0)
          : "memory");
    } else {
      umma_tf32(tmem, ad, bd, idesc, 0);
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float v[32];
  tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), v);
  for (int n = 0; n < 32; ++n) out[(warp * 32 + lane) * 32 + n] = v[n];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
}


// Variant: A K-major (same pattern as B), tf32; or bf16 kind::f16 with both K-major.
template <int BF16>
__global__ void k_mma_k(const float* A, const float* B, float* out) {
  __shared__ __align__(1024) unsigned char sa[4096];
  __shared__ __align__(1024) unsigned char sb[1024];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  for (int idx = tid; idx < 128 * 8; idx += 128) {
    const int m = idx / 8, i = idx % 8;
    if (BF16) {  // 8 bf16 per 16B chunk: K=16 per MMA, i<8 real, 8..15 zero -> only chunk 0
      const int off = (m >> 3) * 256 + (m & 7) * 16 + i * 2;
      *reinterpret_cast<__nv_bfloat16*>(sa + off) = __float2bfloat16(A[m * 8 + i]);
      *reinterpret_cast<__nv_bfloat16*>(sa + off + 128) = __float2bfloat16(0.f);
    } else {
      const int off = (m >> 3) * 256 + ((i >> 2) & 1) * 128 + (m & 7) * 16 + (i & 3) * 4;
      *reinterpret_cast<float*>(sa + off) = A[m * 8 + i];
    }
  }
  for (int idx = tid; idx < 32 * 8; idx += 128) {
    const int nn = idx / 8, i = idx % 8;
    if (BF16) {
      const int off = (nn >> 3) * 256 + (nn & 7) * 16 + i * 2;
      *reinterpret_cast<__nv_bfloat16*>(sb + off) = __float2bfloat16(B[nn * 8 + i]);
      *reinterpret_cast<__nv_bfloat16*>(sb + off + 128) = __float2bfloat16(0.f);
    } else {
      const int off = (nn >> 3) * 256 + ((i >> 2) & 1) * 128 + (nn & 7) * 16 + (i & 3) * 4;
      *reinterpret_cast<float*>(sb + off) = B[nn * 8 + i];
    }
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (tid == 0) {
    const uint64_t ad = umma_desc(smem_u32(sa), 128, 256), bd = umma_desc(smem_u32(sb), 128, 256);
    if (BF16) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                   "l"(ad), "l"(bd), "r"(idesc), "r"(0) : "memory");
    } else {
      const uint32_t idesc = umma_idesc_tf32(128, 32) & ~(1u << 15);
      umma_tf32(tmem, ad, bd, idesc, 0);
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float v[32];
  tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), v);
  for (int n = 0; n < 32; ++n) out[(warp * 32 + lane) * 32 + n] = v[n];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
}


// Variant: A MN-major with SWIZZLE_128B_BASE32B (layout type 1), B K-major, tf32.
__global__ void k_mma_sw(const float* A, const float* B, float* out) {
  __shared__ __align__(1024) unsigned char sa[4096];
  __shared__ __align__(1024) unsigned char sb[1024];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  for (int idx = tid; idx < 8 * 32; idx += 128) {
    const int i = idx / 32, mc = idx % 32;
    const int off = (i >> 2) * 2048 + (mc >> 3) * 512 + (i & 3) * 128 + (((mc & 7) * 16) ^ ((i & 3) << 5));
    float* dst = reinterpret_cast<float*>(sa + off);
    for (int q = 0; q < 4; ++q) dst[q] = A[(4 * mc + q) * 8 + i];
  }
  for (int idx = tid; idx < 32 * 8; idx += 128) {
    const int nn = idx / 8, i = idx % 8;
    const int off = (nn >> 3) * 256 + ((i >> 2) & 1) * 128 + (nn & 7) * 16 + (i & 3) * 4;
    *reinterpret_cast<float*>(sb + off) = B[nn * 8 + i];
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (tid == 0) {
    const uint32_t idesc = umma_idesc_tf32(128, 32);
    const uint64_t ad = umma_desc(smem_u32(sa), 512, 2048) | (1ull << 61), bd = umma_desc(smem_u32(sb), 128, 256);
    umma_tf32(tmem, ad, bd, idesc, 0);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float v[32];
  tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), v);
  for (int n = 0; n < 32; ++n) out[(warp * 32 + lane) * 32 + n] = v[n];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
}

int main() {
  float *d_out, *dA, *dB;
  uint32_t* d_t;
  CK(cudaMalloc(&d_out, 128 * 32 * 4));
  CK(cudaMalloc(&d_t, 4));
  CK(cudaMemset(d_out, 0, 128 * 32 * 4));
  k_roundtrip<<<1, 128>>>(d_out, d_t);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> h(128 * 32);
  uint32_t ta;
  CK(cudaMemcpy(h.data(), d_out, h.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&ta, d_t, 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int t = 0; t < 128; ++t)
    for (int i = 0; i < 32; ++i) bad += h[t * 32 + i] != t * 100 + i;
  printf("roundtrip taddr=0x%08x bad=%d  sample %g %g %g\n", ta, bad, h[0], h[33], h[127 * 32 + 31]);

  std::vector<float> A(128 * 8), B(32 * 8), ref(128 * 32, 0.f);
  for (int m = 0; m < 128; ++m)
    for (int i = 0; i < 8; ++i) A[m * 8 + i] = (float)((m * 3 + i * 5) % 7 - 3);
  for (int n = 0; n < 32; ++n)
    for (int i = 0; i < 8; ++i) B[n * 8 + i] = (float)((n * 2 + i * 3) % 5 - 2);
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 32; ++n)
      for (int i = 0; i < 8; ++i) ref[m * 32 + n] += A[m * 8 + i] * B[n * 8 + i];
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dB, B.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  for (int mask = 0; mask < 5; ++mask) {
    CK(cudaMemset(d_out, 0, 128 * 32 * 4));
    if (mask == 1) k_mma<1><<<1, 128>>>(dA, dB, d_out); else if (mask == 0) k_mma<0><<<1, 128>>>(dA, dB, d_out);
    else if (mask == 2) k_mma_k<0><<<1, 128>>>(dA, dB, d_out); else if (mask == 3) k_mma_k<1><<<1, 128>>>(dA, dB, d_out); else k_mma_sw<<<1, 128>>>(dA, dB, d_out);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h.data(), d_out, h.size() * 4, cudaMemcpyDeviceToHost));
    int nb = 0, nz = 0;
    for (int j = 0; j < 128 * 32; ++j) { nb += fabsf(h[j] - ref[j]) > 1e-3f; nz += h[j] != 0; }
    printf("mma mask=%d bad=%d nonzero=%d\n", mask, nb, nz);
    for (int m = 0; m < 3; ++m) {
      printf(" m=%d gpu:", m);
      for (int n = 0; n < 8; ++n) printf(" %5g", h[m * 32 + n]);
      printf("\n     ref:");
      for (int n = 0; n < 8; ++n) printf(" %5g", ref[m * 32 + n]);
      printf("\n");
    }
  }
  return 0;
}

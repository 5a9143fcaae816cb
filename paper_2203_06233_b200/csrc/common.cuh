// common.cuh -- device-side parameter block and sm_100a primitives shared by the
// STAP kernels (cov.cuh, chol.cuh, apply.cuh, fused.cuh).  Product code: this
// file never includes or mirrors anything from oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace stapk {

// Plan dimensions as the kernels see them (include/stap.h documents each field).
struct KParams {
  int C, T, N, D, R, K, B, S, h;
  float lam;
  int dop_begin, dop_count, bin0, nbins, batch;
  long long cube_stride;  // complex elements per cube in the batch = nbins*C*R
  int y_mc;               // stap_params.out_multicast: Y is an NVLS multicast address
  int y_np;               // stap_params.out_n_peers: extra copies of every Y store ...
  long long y_off[7];     // ... at these byte offsets from the store address (peer-mapped buffers)
};

// Y stores.  With p.y_mc the output pointer is a multicast (NVLS) address: one
// multimem.st writes the value into every rank's copy of the buffer over NVSwitch.
// Otherwise the value is stored at the address and, for each of the p.y_np peer
// offsets, at address + offset (a peer-mapped copy of the same slice): an
// all-gather by unicast stores from the epilogue (include/stap.h out_n_peers).
__device__ __forceinline__ void mm_st(float* a, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void mm_st(float2* a, float2 v) {
  asm volatile("multimem.st.relaxed.sys.global.v2.f32 [%0], {%1, %2};" ::"l"(a), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void mm_st(float4* a, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(a), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w) : "memory");
}
template <class V>
__device__ __forceinline__ void st_y(V* a, V v, const KParams& p) {
  if (p.y_mc) {
    mm_st(a, v);
    return;
  }
  *a = v;
#pragma unroll
  for (int i = 0; i < 7; ++i)
    if (i < p.y_np) *reinterpret_cast<V*>(reinterpret_cast<char*>(a) + p.y_off[i]) = v;
}

// Local row of the cube buffer holding global bin a (a may be outside [0, D)):
// (a - bin0) mod D, non-negative (reading c-3, circular Doppler wrap).
__device__ __forceinline__ int local_bin(const KParams& p, int a) {
  int x = (a - p.bin0) % p.D;
  return x < 0 ? x + p.D : x;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// explicit shared-space float2 access (where the compiler would fall back to generic LD/ST)
__device__ __forceinline__ float2 lds_f2(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_f2(uint32_t a, float2 v) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}

// ---- mbarrier + 1-D bulk async copy (the TMA engine: SASS UBLKCP) ----------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {  // release: prior accesses happen-before
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// try_wait with a suspend-time hint (ns): a waiting thread sleeps in hardware until the phase
// completes (or the hint expires) instead of re-issuing the test, so waiting warps stop taking
// issue slots (measured: cov_tc 566 -> 564 us, medium 450 -> 445 us)
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(10000000u)
      : "memory");
}

// ---- complex helpers (float2 = {re, im}) ----------------------------------
// acc += a * conj(b) -- the HERK inner step of K1/K4: two packed FP32x2 FMAs (SASS
// FFMA2, sm_100), one warp instruction per term for re and im.  Each component sees
// exactly the two fmaf of the scalar form in the same order (b.x term, then b.y term),
// so the result is bit-identical to the scalar form.  Measured: K1 3-5% faster; the
// same packing in the solver and apply loops was neutral or slower (they are not
// FMA-issue-bound), so those keep scalar FMAs.
__device__ __forceinline__ void cmac_conj(float2& acc, float2 a, float2 b) {
  acc = __ffma2_rn(a, make_float2(b.x, b.x), acc);
  acc = __ffma2_rn(make_float2(a.y, -a.x), make_float2(b.y, b.y), acc);
}
// acc += conj(a) * b
__device__ __forceinline__ void cmac_conja(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(-a.y, b.x, acc.y);
}
// acc += conj(w) * z with z as the packed operand and w's parts broadcast (SASS FFMA2
// with a scalar operand and the LO_HI.NP selector: no pair construction); per
// component the same two fmaf, same order as cmac_conja(acc, w, z): bit-identical
__device__ __forceinline__ void cmac_conja2(float2& acc, float2 w, float2 z) {
  acc = __ffma2_rn(z, make_float2(w.x, w.x), acc);
  acc = __ffma2_rn(make_float2(z.y, z.x), make_float2(w.y, -w.y), acc);
}
// FFMA2 forms of the three solver updates: the operand reused across the unrolled
// loop is the packed one (or its LO_HI swap), the other is broadcast; per component the
// same two fmaf in the same order as the scalar forms below (bit-identical).
// acc -= a * conj(b), a packed (L[i][j] over rows), b broadcast (L[l][j])
__device__ __forceinline__ void cmsub_conjb2(float2& acc, float2 a, float2 b) {
  acc = __ffma2_rn(a, make_float2(-b.x, -b.x), acc);
  acc = __ffma2_rn(make_float2(a.y, a.x), make_float2(-b.y, b.y), acc);
}
// acc -= a * b, b packed (y_j[k]), a broadcast (L[i][j])
__device__ __forceinline__ void cmsub2(float2& acc, float2 a, float2 b) {
  acc = __ffma2_rn(b, make_float2(-a.x, -a.x), acc);
  acc = __ffma2_rn(make_float2(b.y, b.x), make_float2(a.y, -a.y), acc);
}
// acc -= conj(a) * b, b packed (v_i[k]), a broadcast (L[i][m])
__device__ __forceinline__ void cmsub_conja2(float2& acc, float2 a, float2 b) {
  acc = __ffma2_rn(b, make_float2(-a.x, -a.x), acc);
  acc = __ffma2_rn(make_float2(b.y, b.x), make_float2(-a.y, a.y), acc);
}
// acc -= a * b
__device__ __forceinline__ void cmsub(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(-a.x, b.x, acc.x);
  acc.x = fmaf(a.y, b.y, acc.x);
  acc.y = fmaf(-a.x, b.y, acc.y);
  acc.y = fmaf(-a.y, b.x, acc.y);
}
// acc -= conj(a) * b
__device__ __forceinline__ void cmsub_conja(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(-a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(-a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
}
// acc -= a * conj(b)
__device__ __forceinline__ void cmsub_conjb(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(-a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(-a.y, b.x, acc.y);
  acc.y = fmaf(a.x, b.y, acc.y);
}

__device__ __forceinline__ bool finite_pos(float x) { return x > 0.0f && x <= 3.402823466e38f; }

}  // namespace stapk

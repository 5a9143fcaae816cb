// apply.cuh -- K3: Y[d][k][r] = w_{d,b(r),k}^H z_{d,r} for every owned bin and range cell.
//
// Method (include/stap.h; reading c-12): z_{d,r}[t*C + c] = X[(d-h+t) mod D][c][r].
//
// Design: every snapshot element is used by exactly one output column (all S
// weights of its unit), so the cube is streamed straight from HBM/L2 with
// coalesced 16-byte loads (2 consecutive range cells per thread), 8 rows in
// flight per thread (a per-unit table of row offsets in shared memory keeps
// the address math out of the loop); the unit's weights -- shared by all
// threads of the unit -- are staged in shared memory transposed to [i][k] so
// that the S weights of one snapshot element are read with broadcast float4
// loads.  A thread keeps SMAX x 2 complex accumulators; stores are 16-byte,
// coalesced along r.
#pragma once
#include "common.cuh"

namespace stapk {

__host__ inline int apply_tpu(int K) { return K / 2 < 128 ? K / 2 : 128; }  // threads per unit
__host__ inline size_t apply_smem_bytes(int N, int SMAX, int units_per_cta) {
  return (size_t)units_per_cta * N * SMAX * 8 + (size_t)units_per_cta * N * 8;
}

// grid.x over groups of `upc` units (unit = ((n*Dl + dl)*B + b)); blockDim = upc * tpu.
// REMOTE: Y stores go through st_y (multicast / peer copies, include/stap.h out_multicast /
// out_n_peers); the plain instantiation compiles to ordinary stores only.
template <int SMAX, bool REMOTE>
__global__ void __launch_bounds__(128) apply_kernel(KParams p, const float2* __restrict__ cube,
                                                     const float2* __restrict__ wts,
                                                     float2* __restrict__ out, int tpu, int upc,
                                                     long long units) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int N = p.N, S = p.S, K = p.K, C = p.C;
  float2* Wt = reinterpret_cast<float2*>(smem);                                        // [upc][N][SMAX]
  long long* rowoff = reinterpret_cast<long long*>(smem + (size_t)upc * N * SMAX * 8);  // [upc][N]
  const int tid = threadIdx.x;
  const long long u0 = (long long)blockIdx.x * upc;

  // stage weights, transposed, zero-padded to SMAX; and the snapshot row offsets
  for (int idx = tid; idx < upc * N * SMAX; idx += blockDim.x) {
    const int uu = idx / (N * SMAX);
    const int rem = idx - uu * N * SMAX;
    const int i = rem / SMAX, k = rem - i * SMAX;
    float2 v = make_float2(0.f, 0.f);
    if (u0 + uu < units && k < S) v = wts[(u0 + uu) * S * N + (long long)k * N + i];
    Wt[idx] = v;
  }
  for (int idx = tid; idx < upc * N; idx += blockDim.x) {
    const int uu = idx / N, i = idx - uu * N;
    long long u = u0 + uu;
    if (u >= units) u = units - 1;
    const int b = (int)(u % p.B);
    const long long nd = u / p.B;
    const int dl = (int)(nd % p.dop_count), n = (int)(nd / p.dop_count);
    const int t = i / C, c = i - t * C;
    const int lb = local_bin(p, p.dop_begin + dl - p.h + t);
    rowoff[idx] = (long long)n * p.cube_stride + ((long long)lb * C + c) * p.R + (long long)b * K;
  }
  __syncthreads();

  const int uu = tid / tpu, tp = tid - uu * tpu;
  const long long u = u0 + uu;
  if (uu >= upc || u >= units) return;
  const int b = (int)(u % p.B);
  const long long nd = u / p.B;  // n*Dl + dl
  const float2* w_s = Wt + (size_t)uu * N * SMAX;
  const long long* ro = rowoff + (size_t)uu * N;
  float2* yb = out + nd * S * p.R + (long long)b * K;

  for (int jp = tp; jp < K / 2; jp += tpu) {
    const int j = 2 * jp;
    float2 acc0[SMAX], acc1[SMAX];
#pragma unroll
    for (int k = 0; k < SMAX; ++k) acc0[k] = acc1[k] = make_float2(0.f, 0.f);
    for (int i0 = 0; i0 < N; i0 += 8) {
      float4 z[8];
#pragma unroll
      for (int v = 0; v < 8; ++v)
        z[v] = (i0 + v < N) ? __ldg(reinterpret_cast<const float4*>(cube + ro[i0 + v] + j))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        if (i0 + v < N) {
          const float2 z0 = make_float2(z[v].x, z[v].y), z1 = make_float2(z[v].z, z[v].w);
          const float4* wv = reinterpret_cast<const float4*>(w_s + (i0 + v) * SMAX);
#pragma unroll
          for (int k2 = 0; k2 < SMAX / 2; ++k2) {
            const float4 ww = wv[k2];
            cmac_conja2(acc0[2 * k2], make_float2(ww.x, ww.y), z0);
            cmac_conja2(acc1[2 * k2], make_float2(ww.x, ww.y), z1);
            cmac_conja2(acc0[2 * k2 + 1], make_float2(ww.z, ww.w), z0);
            cmac_conja2(acc1[2 * k2 + 1], make_float2(ww.z, ww.w), z1);
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < SMAX; ++k)
      if (k < S) {
        float4* ya = reinterpret_cast<float4*>(yb + (long long)k * p.R + j);
        const float4 yv = make_float4(acc0[k].x, acc0[k].y, acc1[k].x, acc1[k].y);
        if constexpr (REMOTE) st_y(ya, yv, p);
        else *ya = yv;
      }
  }
}

}  // namespace stapk

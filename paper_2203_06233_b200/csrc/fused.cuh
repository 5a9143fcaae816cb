// fused.cuh -- K4: the whole path in one kernel (stap_run): cube in, Y out,
// no HBM intermediates.
//
// Method: exactly K1 -> K2 -> K3 (cov.cuh, solve.cuh, apply.cuh) for every unit;
// the same device functions compute the lag blocks, the loaded covariance and
// the warp-level Cholesky/solves, so a fused unit is computed with the same
// summation orders as the staged path.
//
// One CTA owns (run of P bins, training block b, cube n):
//   1. warp 0 bulk-copies the W = P+T-1 bin window of block b into shared
//      memory (TMA engine, one mbarrier); the other warps stage the steering set;
//   2. one thread per lag block (w, w+l): C x C HERK over the K cells -> shared;
//   3. delta per bin from the lag-0 blocks;
//   4. warps take bins round-robin: assemble the loaded R (lower triangle),
//      Cholesky + solves (warp_chol_solve) -> w_k in shared [i][k], then apply
//      the S weights to the K cells of the bin straight from the window
//      (lane = range cell, S accumulators, broadcast float4 weight reads) and
//      store Y with coalesced 8-byte stores.
// Chosen when it fits in <= 113 KB of shared memory with >= 4 warps (2 CTAs/SM);
// otherwise stap_run runs the staged K1 -> K2 -> K3.
#pragma once
#include <cstdio>
#include <cstring>

#include "cov.cuh"
#include "solve.cuh"

namespace stapk {

struct FusedCfg {
  int C, SMAX, P, threads, runs;
  size_t smem;
  char name[96];
};

__host__ __device__ inline size_t fused_off_blk(int C, int T, int K, int P) {
  return (((size_t)(P + T - 1) * cov_binstride(C, K) * 8) + 15) & ~(size_t)15;
}
__host__ __device__ inline size_t fused_off_warps(int C, int T, int K, int P) {
  return fused_off_blk(C, T, K, P) + (((size_t)cov_blocks(T, P + T - 1) * C * C * 8 + 15) & ~(size_t)15);
}
__host__ __device__ inline size_t fused_warp_bytes(int N, int SMAX) {
  return (((size_t)N * solve_ld(N) + (size_t)N * SMAX) * 8 + 15) & ~(size_t)15;
}
__host__ __device__ inline size_t fused_off_steer(int C, int T, int K, int P, int N, int SMAX, int nw) {
  return fused_off_warps(C, T, K, P) + (size_t)nw * fused_warp_bytes(N, SMAX);
}
__host__ __device__ inline size_t fused_off_bar(int C, int T, int K, int P, int N, int S, int SMAX, int nw) {
  return fused_off_steer(C, T, K, P, N, SMAX, nw) + ((((size_t)S * N * 8) + 15) & ~(size_t)15);
}
__host__ inline size_t fused_smem_bytes(int C, int T, int K, int P, int N, int S, int SMAX, int nw) {
  return fused_off_bar(C, T, K, P, N, S, SMAX, nw) + 16 + (size_t)P * 4;
}

template <int C, int SMAX>
__global__ void __launch_bounds__(256) fused_kernel(KParams p, const float2* __restrict__ cube,
                                                     const float2* __restrict__ steer, float2* __restrict__ out,
                                                     int32_t* __restrict__ info, int P) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int run = blockIdx.x, b = blockIdx.y, n = blockIdx.z;
  const int T = p.T, K = p.K, N = p.N, S = p.S;
  const int nw = blockDim.x >> 5;
  const int dl0 = run * P;
  const int Prun = min(P, p.dop_count - dl0);
  const int d0 = p.dop_begin + dl0;
  const int W = Prun + T - 1;
  const int nblk = cov_blocks(T, W);
  const int bstride = cov_binstride(C, K);
  const int LD = solve_ld(N);

  float2* xs = reinterpret_cast<float2*>(smem);
  float2* blk = reinterpret_cast<float2*>(smem + fused_off_blk(C, T, K, P));
  unsigned char* wbase = smem + fused_off_warps(C, T, K, P);
  float2* steer_s = reinterpret_cast<float2*>(smem + fused_off_steer(C, T, K, P, N, SMAX, nw));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + fused_off_bar(C, T, K, P, N, S, SMAX, nw));
  float* delta_s = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(bar) + 16);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float2* L = reinterpret_cast<float2*>(wbase + (size_t)warp * fused_warp_bytes(N, SMAX));
  float2* Y = L + (size_t)N * LD;  // [N][SMAX]

  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) {
    load_window(p, cube, n, b, d0, W, C, bstride, xs, bar);
  } else {
    for (int idx = tid - 32; idx < S * N; idx += blockDim.x - 32) steer_s[idx] = steer[idx];
  }
  for (int idx = lane; idx < N * SMAX; idx += 32) Y[idx] = make_float2(0.f, 0.f);  // zero padding columns

  // 2. lag-block HERK
  {
    int w, l;
    lag_block_of(tid, T, W, w, l);
    mbar_wait(bar, 0);
    if (tid < nblk) {
      float2 acc[C][C];
      herk_block<C>(xs + w * bstride, xs + (w + l) * bstride, K, acc);
      const float invK = 1.0f / (float)K;
#pragma unroll
      for (int c = 0; c < C; ++c)
#pragma unroll
        for (int c2 = 0; c2 < C; ++c2)
          blk[(tid * C + c) * C + c2] = make_float2(acc[c][c2].x * invK, acc[c][c2].y * invK);
    }
  }
  __syncthreads();
  if (tid < Prun) delta_s[tid] = delta_from_blocks(blk, C, T, N, p.lam, tid);
  __syncthreads();

  // 4. per bin: loaded R -> Cholesky + solves -> apply
  for (int pr = warp; pr < Prun; pr += nw) {
    const float dlt = delta_s[pr];
    for (int idx = lane; idx < N * N; idx += 32) {
      const int i = idx / N, col = idx - i * N;
      if (col > i) continue;
      float2 v = rhat_from_blocks(blk, C, W, pr, i, col);
      if (i == col) {
        v.y = 0.f;
        v.x += dlt;
      }
      L[i * LD + col] = v;
    }
    __syncwarp();
    float g = 0.f;
    const int inf = warp_chol_solve(N, S, SMAX, L, Y, steer_s, &g);
    const int dl = dl0 + pr;
    if (lane == 0) info[((long long)n * p.dop_count + dl) * p.B + b] = inf;

    float2* yb = out + (((long long)n * p.dop_count + dl) * S) * p.R + (long long)b * K;
    const float2* xw = xs + pr * bstride;
    for (int j = lane; j < K; j += 32) {
      float2 acc[SMAX];
#pragma unroll
      for (int k = 0; k < SMAX; ++k) acc[k] = make_float2(0.f, 0.f);
      int i = 0;
      for (int t = 0; t < T; ++t) {
        for (int c = 0; c < C; ++c, ++i) {
          const float2 z = xw[t * bstride + c * K + j];
          const float4* wv = reinterpret_cast<const float4*>(Y + i * SMAX);
#pragma unroll
          for (int k2 = 0; k2 < SMAX / 2; ++k2) {
            const float4 ww = wv[k2];
            cmac_conja(acc[2 * k2], make_float2(ww.x, ww.y), z);
            cmac_conja(acc[2 * k2 + 1], make_float2(ww.z, ww.w), z);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < SMAX; ++k)
        if (k < S) yb[(long long)k * p.R + j] = acc[k];
    }
    __syncwarp();
  }
}

// ---- host-side selection / launch ------------------------------------------
template <int C, int SMAX>
inline void fused_launch_t(const FusedCfg& f, const KParams& kp, const float2* cube, const float2* steer,
                           float2* out, int32_t* info, cudaStream_t st) {
  dim3 grid(f.runs, kp.B, kp.batch);
  fused_kernel<C, SMAX><<<grid, f.threads, f.smem, st>>>(kp, cube, steer, out, info, f.P);
}
template <int C, int SMAX>
inline void fused_attr_t(const FusedCfg& f) {
  cudaFuncSetAttribute(fused_kernel<C, SMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f.smem);
}

#define STAPK_FUSED_DISPATCH(FN, ...)                                   \
  switch (f.C * 100 + f.SMAX) {                                         \
    case 102: FN<1, 2>(__VA_ARGS__); break;                             \
    case 104: FN<1, 4>(__VA_ARGS__); break;                             \
    case 108: FN<1, 8>(__VA_ARGS__); break;                             \
    case 116: FN<1, 16>(__VA_ARGS__); break;                            \
    case 132: FN<1, 32>(__VA_ARGS__); break;                            \
    case 202: FN<2, 2>(__VA_ARGS__); break;                             \
    case 204: FN<2, 4>(__VA_ARGS__); break;                             \
    case 208: FN<2, 8>(__VA_ARGS__); break;                             \
    case 216: FN<2, 16>(__VA_ARGS__); break;                            \
    case 232: FN<2, 32>(__VA_ARGS__); break;                            \
    case 302: FN<3, 2>(__VA_ARGS__); break;                             \
    case 304: FN<3, 4>(__VA_ARGS__); break;                             \
    case 308: FN<3, 8>(__VA_ARGS__); break;                             \
    case 316: FN<3, 16>(__VA_ARGS__); break;                            \
    case 332: FN<3, 32>(__VA_ARGS__); break;                            \
    case 402: FN<4, 2>(__VA_ARGS__); break;                             \
    case 404: FN<4, 4>(__VA_ARGS__); break;                             \
    case 408: FN<4, 8>(__VA_ARGS__); break;                             \
    case 416: FN<4, 16>(__VA_ARGS__); break;                            \
    case 432: FN<4, 32>(__VA_ARGS__); break;                            \
    case 602: FN<6, 2>(__VA_ARGS__); break;                             \
    case 604: FN<6, 4>(__VA_ARGS__); break;                             \
    case 608: FN<6, 8>(__VA_ARGS__); break;                             \
    case 616: FN<6, 16>(__VA_ARGS__); break;                            \
    case 632: FN<6, 32>(__VA_ARGS__); break;                            \
    case 802: FN<8, 2>(__VA_ARGS__); break;                             \
    case 804: FN<8, 4>(__VA_ARGS__); break;                             \
    case 808: FN<8, 8>(__VA_ARGS__); break;                             \
    case 816: FN<8, 16>(__VA_ARGS__); break;                            \
    case 832: FN<8, 32>(__VA_ARGS__); break;                            \
    default: break;                                                     \
  }

inline bool fused_supported_C(int C) { return C == 1 || C == 2 || C == 3 || C == 4 || C == 6 || C == 8; }

// Pick (P, threads) for the fused kernel; false -> use the staged path.
inline bool fused_configure(const KParams& kp, FusedCfg* f) {
  memset(f, 0, sizeof *f);
  if (!fused_supported_C(kp.C)) return false;
  const int S = kp.S;
  const int SMAX = S <= 2 ? 2 : S <= 4 ? 4 : S <= 8 ? 8 : S <= 16 ? 16 : 32;
  const size_t cap = 113 * 1024;
  for (int threads = 128; threads <= 256; threads += 128) {
    const int nw = threads / 32;
    for (int P = kp.dop_count < 64 ? kp.dop_count : 64; P >= 1; --P) {
      if (cov_blocks(kp.T, P + kp.T - 1) > threads) continue;
      const size_t sm = fused_smem_bytes(kp.C, kp.T, kp.K, P, kp.N, S, SMAX, nw);
      if (sm > cap) continue;
      f->C = kp.C;
      f->SMAX = SMAX;
      f->P = P;
      f->threads = threads;
      f->runs = (kp.dop_count + P - 1) / P;
      f->smem = sm;
      snprintf(f->name, sizeof f->name, "C=%d,SMAX=%d,P=%d,threads=%d,smem=%zu", kp.C, SMAX, P, threads, sm);
      return true;
    }
  }
  return false;
}

inline void fused_set_attr(const FusedCfg& f) { STAPK_FUSED_DISPATCH(fused_attr_t, f) }

inline void fused_launch(const FusedCfg& f, const KParams& kp, const float2* cube, const float2* steer,
                         float2* out, int32_t* info, cudaStream_t st) {
  STAPK_FUSED_DISPATCH(fused_launch_t, f, kp, cube, steer, out, info, st)
}

}  // namespace stapk

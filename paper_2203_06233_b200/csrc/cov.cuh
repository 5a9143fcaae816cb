// cov.cuh -- K1: loaded covariance of every owned unit (d, b).
//
// Method (include/stap.h; readings c-2..c-7): for unit (d, b) the
// snapshot rows are z[t*C + c][j] = X[(d-h+t) mod D][c][bK + j] and
//   Rhat[i][l] = (1/K) sum_j z[i][j] conj(z[l][j]),  R = Rhat + (lambda tr(Rhat)/N) I.
//
// B200 design -- Doppler-lag block sharing: the (t, t')
// C x C block of R_d is P(a, a') = (1/K) sum_j x_a[.][j] x_a'[.][j]^H with
// a = d-h+t, a' = d-h+t', so a CTA that owns a run of P consecutive bins of one
// training block computes every lag block (w, w+l), l < T, of its window of
// W = P+T-1 bins ONCE and assembles the P matrices from them: T*W - T(T-1)/2
// blocks instead of P*T(T+1)/2.  Each block's sum runs over j in ascending
// order no matter which CTA computes it, so the result is bitwise independent
// of P, of the run alignment and of the Doppler shard.
//
// Staging: the window (W bins x C channels x K cells, each row K*8 contiguous
// bytes in HBM) is copied to shared memory with 1-D bulk async copies (TMA
// engine) completing on one mbarrier.  Shared layout [w][c][j] with a 16-byte
// pad per bin, so lanes reading the same (c, j) of 8 consecutive bins hit 8
// distinct 16-byte bank groups.  One thread owns one lag block: C x C complex
// accumulators in registers, float4 (2 cells) loads along j.
#pragma once
#include "common.cuh"

namespace stapk {

__host__ __device__ inline int cov_blocks(int T, int W) { return T * W - T * (T - 1) / 2; }
__host__ __device__ inline int cov_binstride(int C, int K) { return C * K + 2; }  // complex
__host__ inline size_t cov_smem_bytes(int C, int T, int K, int P) {
  const int W = P + T - 1;
  size_t win = (size_t)W * cov_binstride(C, K) * 8;
  size_t blk = (size_t)cov_blocks(T, W) * C * C * 8;
  size_t body = win > blk ? win : blk;
  body = (body + 15) & ~(size_t)15;
  return body + 16 /*mbarrier*/ + (size_t)P * 4 /*delta*/ + 16;
}


// Issue the bulk copies of a window of W bins (global bins d0-h .. d0-h+W-1,
// wrapped) of training block b of cube n into xs[w*bstride + c*K + j]; one
// mbarrier `bar` (initialised with count 1) completes when all bytes landed.
// Called by warp 0 only.
__device__ __forceinline__ void load_window(const KParams& p, const float2* __restrict__ cube, int n, int b,
                                            int d0, int W, int C, int bstride, float2* xs, uint64_t* bar) {
  const int lane = threadIdx.x & 31, K = p.K;
  if (lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)(W * C * K * 8));
  __syncwarp();
  const float2* cb = cube + (long long)n * p.cube_stride + (long long)b * K;
  for (int q = lane; q < W * C; q += 32) {
    const int w = q / C, c = q - w * C;
    const int lb = local_bin(p, d0 - p.h + w);
    bulk_g2s(xs + w * bstride + c * K, cb + ((long long)lb * C + c) * p.R, (uint32_t)(K * 8), bar);
  }
}

// Lag-major block enumeration: block index t -> (w, l), block (w, w+l), w < W - l.
__device__ __forceinline__ void lag_block_of(int t, int T, int W, int& w, int& l) {
  l = 0;
  w = t;
  while (l < T && w >= W - l) {
    w -= W - l;
    ++l;
  }
}
__host__ __device__ inline int lag_block_index(int w, int l, int W) { return l * W - l * (l - 1) / 2 + w; }

// acc[c][c2] = sum_j xa[c][j] conj(xb[c2][j]), j ascending (fixed order).
template <int C>
__device__ __forceinline__ void herk_block(const float2* xa, const float2* xb, int K, float2 (&acc)[C][C]) {
#pragma unroll
  for (int c = 0; c < C; ++c)
#pragma unroll
    for (int c2 = 0; c2 < C; ++c2) acc[c][c2] = make_float2(0.f, 0.f);
#pragma unroll 2
  for (int j = 0; j < K; j += 2) {
    float4 a[C];
#pragma unroll
    for (int c = 0; c < C; ++c) a[c] = *reinterpret_cast<const float4*>(xa + c * K + j);
#pragma unroll
    for (int c2 = 0; c2 < C; ++c2) {
      const float4 bb = *reinterpret_cast<const float4*>(xb + c2 * K + j);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        cmac_conj(acc[c][c2], make_float2(a[c].x, a[c].y), make_float2(bb.x, bb.y));
        cmac_conj(acc[c][c2], make_float2(a[c].z, a[c].w), make_float2(bb.z, bb.w));
      }
    }
  }
}

// Element (i, l) of Rhat for bin p of a run from the scaled lag blocks blk[nblk][C][C]:
// upper (t_i, c_i) <= (t_l, c_l) read directly, lower = conj of the mirrored upper.
__device__ __forceinline__ float2 rhat_from_blocks(const float2* blk, int C, int W, int pr, int i, int col) {
  const int ti = i / C, ci = i - ti * C, tl = col / C, cl = col - tl * C;
  if (ti < tl || (ti == tl && ci <= cl)) {
    return blk[(lag_block_index(pr + ti, tl - ti, W) * C + ci) * C + cl];
  }
  const float2 u = blk[(lag_block_index(pr + tl, ti - tl, W) * C + cl) * C + ci];
  return make_float2(u.x, -u.y);
}

// delta of bin pr: lambda * sum_{i ascending} Re Rhat[i][i] / N  (lag-0 block of bin w is index w).
__device__ __forceinline__ float delta_from_blocks(const float2* blk, int C, int T, int N, float lam, int pr) {
  float tr = 0.f;
  for (int t = 0; t < T; ++t)
    for (int c = 0; c < C; ++c) tr += blk[((pr + t) * C + c) * C + c].x;
  return lam * tr / (float)N;
}

template <int C>
__global__ void __launch_bounds__(256) cov_kernel(KParams p, const float2* __restrict__ cube,
                                                   float2* __restrict__ cov, int P) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int run = blockIdx.x, b = blockIdx.y, n = blockIdx.z;
  const int T = p.T, K = p.K, N = p.N;
  const int dl0 = run * P;                       // first owned (local) bin of this run
  const int Prun = min(P, p.dop_count - dl0);
  const int d0 = p.dop_begin + dl0;              // its global index
  const int W = Prun + T - 1;
  const int nblk = cov_blocks(T, W);
  const int bstride = cov_binstride(C, K);

  float2* xs = reinterpret_cast<float2*>(smem);
  const int Wmax = P + T - 1;
  size_t body = (size_t)Wmax * bstride * 8;
  size_t blkb = (size_t)cov_blocks(T, Wmax) * C * C * 8;
  body = ((body > blkb ? body : blkb) + 15) & ~(size_t)15;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + body);
  float* delta_s = reinterpret_cast<float*>(smem + body + 16);

  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid < 32) load_window(p, cube, n, b, d0, W, C, bstride, xs, bar);

  int w, l;
  lag_block_of(tid, T, W, w, l);
  const bool active = tid < nblk;
  float2 acc[C][C];
  mbar_wait(bar, 0);
  if (active) herk_block<C>(xs + w * bstride, xs + (w + l) * bstride, K, acc);
  __syncthreads();  // window no longer read: reuse the space for the blocks

  const float invK = 1.0f / (float)K;
  float2* blk = reinterpret_cast<float2*>(smem);  // [nblk][C][C], already scaled by 1/K
  if (active) {
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
      for (int c2 = 0; c2 < C; ++c2)
        blk[(tid * C + c) * C + c2] = make_float2(acc[c][c2].x * invK, acc[c][c2].y * invK);
  }
  __syncthreads();

  // delta per bin of the run: lambda * tr(Rhat) / N, trace summed over i = t*C + c ascending.
  // Lag-0 block of window bin w is block index w.
  if (tid < Prun) delta_s[tid] = delta_from_blocks(blk, C, T, N, p.lam, tid);
  __syncthreads();

  // Assemble R_d for each bin of the run (both triangles; lower = conj of upper).
  const long long NN = (long long)N * N;
  float2* out = cov + (((long long)n * p.dop_count + dl0) * p.B + b) * NN;
  const long long ostride = (long long)p.B * NN;  // between consecutive bins
  const int total = Prun * N * N;
  for (int idx = tid; idx < total; idx += blockDim.x) {
    const int pr = idx / (N * N);
    const int rem = idx - pr * N * N;
    const int i = rem / N, col = rem - i * N;
    float2 v = rhat_from_blocks(blk, C, W, pr, i, col);
    if (i == col) {
      v.y = 0.f;
      v.x += delta_s[pr];
    }
    out[pr * ostride + rem] = v;
  }
}

}  // namespace stapk

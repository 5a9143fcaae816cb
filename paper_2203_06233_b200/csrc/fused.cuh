// fused.cuh -- K4: the whole path in one kernel (stap_run): cube in, Y out,
// no HBM intermediates.
//
// Method: exactly K1 -> K2 -> K3 (cov.cuh, solve.cuh, apply.cuh) for every unit;
// the same device functions compute the lag blocks, the loaded covariance and
// the group Cholesky/solves, so a fused unit is computed with the same
// summation orders as the staged path.
//
// One CTA owns (run of P bins, training block b, cube n):
//   1. warp 0 bulk-copies the W = P+T-1 bin window of block b into shared
//      memory (TMA engine, one mbarrier);
//   2. one thread per lag block (w, w+l): C x C HERK over the K cells -> shared;
//   3. delta per bin from the lag-0 blocks;
//   4. solve groups (solve.cuh layout) take bins round-robin: load the loaded R
//      straight from the lag blocks into registers, Cholesky + solves, publish
//      w_k in shared [i][SMAX], then apply the S weights to the K cells of the
//      bin straight from the window (lane = range cell, S accumulators,
//      broadcast float4 weight reads) and store Y with coalesced 8-byte stores.
// Instantiated for the BASELINE.json shapes; other shapes run the staged path.
#pragma once
#include <cstdio>
#include <cstring>

#include "cov.cuh"
#include "solve.cuh"

namespace stapk {

struct FusedCfg {
  int C, SMAX, solve_id, P, threads, runs;
  size_t smem;
  char name[112];
};

struct FusedLayout {
  size_t off_blk, off_sh, off_w, off_bar, total;
};

__host__ __device__ inline FusedLayout fused_layout(int C, int T, int K, int P, int N, int SMAX, int ngroups,
                                                    size_t sh_bytes) {
  FusedLayout L;
  size_t o = (((size_t)(P + T - 1) * cov_binstride(C, K) * 8) + 127) & ~(size_t)127;
  L.off_blk = o;
  o += (((size_t)cov_blocks(T, P + T - 1) * C * C * 8) + 127) & ~(size_t)127;
  L.off_sh = o;
  o += ((ngroups * sh_bytes) + 127) & ~(size_t)127;
  L.off_w = o;
  o += (((size_t)ngroups * N * SMAX * 8) + 127) & ~(size_t)127;
  L.off_bar = o;
  L.total = o + 16 + (size_t)P * 4;
  return L;
}

template <int C, int SMAX, class CF>
__global__ void __launch_bounds__(256) fused_kernel(KParams p, const float2* __restrict__ cube,
                                                     const float2* __restrict__ steer, float2* __restrict__ out,
                                                     int32_t* __restrict__ info, int P) {
  constexpr int G = CF::G, PR = CF::PR, PC = CF::PC, MR = CF::MR, MC = CF::MC, SC = CF::SC;
  extern __shared__ __align__(128) unsigned char smem[];
  const int run = blockIdx.x, b = blockIdx.y, n = blockIdx.z;
  const int T = p.T, K = p.K, N = p.N, S = p.S;
  const int ngroups = blockDim.x / G;
  const int dl0 = run * P;
  const int Prun = min(P, p.dop_count - dl0);
  const int d0 = p.dop_begin + dl0;
  const int W = Prun + T - 1;
  const int nblk = cov_blocks(T, W);
  const int bstride = cov_binstride(C, K);
  const FusedLayout lay = fused_layout(C, T, K, P, N, SMAX, ngroups, sizeof(SolveShared<CF>));

  float2* xs = reinterpret_cast<float2*>(smem);
  float2* blk = reinterpret_cast<float2*>(smem + lay.off_blk);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + lay.off_bar);
  float* delta_s = reinterpret_cast<float*>(smem + lay.off_bar + 16);

  const int tid = threadIdx.x;
  const int grp = tid / G, gl = tid - grp * G;
  const int gp = gl / PC, gq = gl - (gl / PC) * PC;
  SolveShared<CF>& sh = reinterpret_cast<SolveShared<CF>*>(smem + lay.off_sh)[grp];
  float2* wsm = reinterpret_cast<float2*>(smem + lay.off_w) + (size_t)grp * N * SMAX;  // [N][SMAX]
  const int bar_id = 1 + grp;

  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid < 32) load_window(p, cube, n, b, d0, W, C, bstride, xs, bar);
  for (int idx = gl; idx < N * SMAX; idx += G) wsm[idx] = make_float2(0.f, 0.f);  // zero padding columns

  // 2. lag-block HERK, one thread per block
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

  // 4. bins round-robin over the solve groups (trip count uniform per warp)
  constexpr int GPW = G < 32 ? 32 / G : 1;
  const int wg0 = (grp / GPW) * GPW;
  for (int base = wg0; base < Prun; base += ngroups) {
    const int pr_raw = base + (grp - wg0);
    const bool valid = pr_raw < Prun;
    const int pr = valid ? pr_raw : Prun - 1;
    const float dlt = delta_s[pr];
    float2 A[MR][MC], B[MR][SC];
#pragma unroll
    for (int v = 0; v < MC; ++v)
#pragma unroll
      for (int u = CF::umin(v); u < MR; ++u) {
        const int i = PR * u + gp, l = PC * v + gq;
        float2 x = make_float2(0.f, 0.f);
        if (i < N && l <= i) {
          x = rhat_from_blocks(blk, C, W, pr, i, l);
          if (i == l) x = make_float2(x.x + dlt, 0.f);
        }
        A[u][v] = x;
      }
#pragma unroll
    for (int u = 0; u < MR; ++u)
#pragma unroll
      for (int kv = 0; kv < SC; ++kv) {
        const int i = PR * u + gp, k = PC * kv + gq;
        B[u][kv] = (i < N && k < S) ? __ldg(steer + k * N + i) : make_float2(0.f, 0.f);
      }
    const int inf = group_chol_solve<CF>(N, S, A, B, sh, gl, bar_id);
#pragma unroll
    for (int u = 0; u < MR; ++u)
#pragma unroll
      for (int kv = 0; kv < SC; ++kv) {
        const int i = PR * u + gp, k = PC * kv + gq;
        if (i < N && k < S) wsm[i * SMAX + k] = B[u][kv];
      }
    group_sync<G>(bar_id);

    const int dl = dl0 + pr;
    if (valid) {
      if (gl == 0) info[((long long)n * p.dop_count + dl) * p.B + b] = inf;
      float2* yb = out + (((long long)n * p.dop_count + dl) * S) * p.R + (long long)b * K;
      const float2* xw = xs + pr * bstride;
      for (int j = gl; j < K; j += G) {
        float2 acc[SMAX];
#pragma unroll
        for (int k = 0; k < SMAX; ++k) acc[k] = make_float2(0.f, 0.f);
        int i = 0;
        for (int t = 0; t < T; ++t) {
          for (int c = 0; c < C; ++c, ++i) {
            const float2 z = xw[t * bstride + c * K + j];
            const float4* wv = reinterpret_cast<const float4*>(wsm + i * SMAX);
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
    }
    group_sync<G>(bar_id);
  }
}

// ---- host-side selection / launch ------------------------------------------
// (C, SMAX, solve config id) instantiations: the BASELINE.json shapes.
#define STAPK_FUSED_CFGS(X) \
  X(2, 4, 0, SolveCfg0)        \
  X(4, 16, 6, SolveCfg6)       \
  X(6, 16, 16, SolveCfg16)     \
  X(8, 16, 22, SolveCfg22)

inline int fused_smax(int S) { return S <= 2 ? 2 : S <= 4 ? 4 : S <= 8 ? 8 : S <= 16 ? 16 : 32; }

// Pick (P, threads) for the fused kernel; false -> use the staged path.
inline bool fused_configure(const KParams& kp, FusedCfg* f) {
  memset(f, 0, sizeof *f);
  SolveSel sel;
  if (!solve_select(kp.N, kp.S, &sel)) return false;
  const int SMAX = fused_smax(kp.S);
  bool have = false;
#define X(CC, SM, ID, CFT) \
  if (kp.C == CC && SMAX == SM && sel.id == ID) have = true;
  STAPK_FUSED_CFGS(X)
#undef X
  if (!have) return false;
  const size_t cap = 227 * 1024;
  int bestP = 0, bestT = 0;
  size_t bestS = 0;
  double bestScore = -1.0;
  for (int threads = 128; threads <= 256; threads += 128) {
    if (threads % sel.G) continue;
    const int ng = threads / sel.G;
    for (int P = 1; P <= kp.dop_count && P <= 64; ++P) {
      if (cov_blocks(kp.T, P + kp.T - 1) > threads) break;
      const FusedLayout L = fused_layout(kp.C, kp.T, kp.K, P, kp.N, SMAX, ng, sel.shared_bytes);
      if (L.total > cap) break;
      const int cta_per_sm = (int)((228 * 1024) / (L.total + 1024));
      const int warps = cta_per_sm * threads / 32;
      if (cta_per_sm < 1) break;
      // prefer more resident warps, then less covariance work per bin (larger P)
      const double score = (warps > 16 ? 16 : warps) * 1000.0 + P;
      if (score > bestScore) {
        bestScore = score;
        bestP = P;
        bestT = threads;
        bestS = L.total;
      }
    }
  }
  if (bestP == 0) return false;
  f->C = kp.C;
  f->SMAX = SMAX;
  f->solve_id = sel.id;
  f->P = bestP;
  f->threads = bestT;
  f->runs = (kp.dop_count + bestP - 1) / bestP;
  f->smem = bestS;
  snprintf(f->name, sizeof f->name, "C=%d,SMAX=%d,solve=%d(G=%d),P=%d,threads=%d,smem=%zu", kp.C, SMAX, sel.id,
           sel.G, bestP, bestT, bestS);
  return true;
}

inline void fused_set_attr(const FusedCfg& f) {
#define X(CC, SM, ID, CFT)                                                                                   \
  if (f.C == CC && f.SMAX == SM && f.solve_id == ID)                                                        \
    cudaFuncSetAttribute(fused_kernel<CC, SM, CFT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f.smem);
  STAPK_FUSED_CFGS(X)
#undef X
}

inline void fused_launch(const FusedCfg& f, const KParams& kp, const float2* cube, const float2* steer,
                         float2* out, int32_t* info, cudaStream_t st) {
  dim3 grid(f.runs, kp.B, kp.batch);
#define X(CC, SM, ID, CFT)                              \
  if (f.C == CC && f.SMAX == SM && f.solve_id == ID)   \
    fused_kernel<CC, SM, CFT><<<grid, f.threads, f.smem, st>>>(kp, cube, steer, out, info, f.P);
  STAPK_FUSED_CFGS(X)
#undef X
}

}  // namespace stapk

// fused.cuh -- K4: the whole path in one kernel (stap_run): cube in, Y out,
// no HBM intermediates.
//
// Method: exactly K1 -> K2 -> K3 (cov.cuh, chol.cuh / solve_small.cuh,
// apply.cuh) for every unit; the same device functions compute the lag
// blocks, the loaded covariance and the Cholesky/solves, so a fused unit is
// computed with the same summation orders as the staged path.
//
// One CTA owns (run of P bins, training block b, cube n):
//   1. warp 0 bulk-copies the W = P+T-1 bin window of block b into shared
//      memory (TMA engine, one mbarrier), layout [w][c][K+2] (+ bin pad);
//   2. lag-block HERK (cta_lag_blocks) -> scaled blocks in shared memory;
//   3. delta per bin from the lag-0 blocks;
//   4. solver segments (a lane group per matrix) take bins round-robin: load the
//      loaded R straight from the lag blocks into registers, Cholesky + solves
//      (solve_small.cuh for N = 12 and below, chol.cuh above),
//      publish w_k in shared [i][SMAX], then apply the S weights to the K cells
//      of the bin straight from the window (lane = range cell, S accumulators,
//      broadcast float4 weight reads) and store Y with coalesced 8-byte stores.
// Instantiated for the BASELINE.json shapes; other shapes run the staged path.
#pragma once
#include <cstdio>
#include <cstring>

#include "cov.cuh"
#include "chol.cuh"
#include "solve_small.cuh"

namespace stapk {

#ifdef STAPK_PROF
// phase-cycle counters of the fused kernel (profiling builds only):
// [0] lag-block HERK + delta (per CTA), [1] solves (per segment), [2] apply (per segment), [3] CTA total
__device__ unsigned long long g_fused_prof[4];
#define STAPK_PROF_T(v) const long long v = clock64()
#define STAPK_PROF_ADD(i, x) atomicAdd(&g_fused_prof[i], (unsigned long long)(x))
#else
#define STAPK_PROF_T(v)
#define STAPK_PROF_ADD(i, x)
#endif

struct FusedCfg {
  int C, SMAX, N, G, P, threads, runs;
  size_t smem;
  char name[112];
};

struct FusedLayout {
  size_t off_blk, off_sh, off_w, off_bar, total;
};

__host__ __device__ inline FusedLayout fused_layout(int C, int T, int K, int P, int N, int SMAX, int ngroups,
                                                    size_t sh_bytes) {
  FusedLayout L;
  size_t o = (((size_t)(P + T - 1) * tile_bs(C, K) * 8) + 127) & ~(size_t)127;  // whole window, KC = K
  L.off_blk = o;
  o += (((size_t)cov_blocks(T, P + T - 1) * blk_stride(C) * 8) + 127) & ~(size_t)127;
  L.off_sh = o;
  o += ((ngroups * sh_bytes) + 127) & ~(size_t)127;
  L.off_w = o;
  o += (((size_t)ngroups * N * SMAX * 8) + 127) & ~(size_t)127;
  L.off_bar = o;
  L.total = o + 16 + (size_t)P * 4;
  return L;
}

// ---- solver policies: load R of bin pr from the lag blocks, solve, publish w in wsm[i][SMAX]
template <class CF>
struct CholSolverPolicy {
  static constexpr int G = CF::G;
  static constexpr int kMaxThreads = 256, kMinBlocks = CF::G > 32 ? 1 : 2;
  static constexpr bool kWInShared = false;
  static constexpr int kN = 0;
  using Shared = CholShared<CF>;
  template <int C, int SMAX>
  __device__ static __forceinline__ int solve_bin(const KParams& p, const float2* blk, int W, int pr, float dlt,
                                                  const float2* __restrict__ steer, Shared& sh, int gl, int bar_id,
                                                  float2* wsm) {
    constexpr int PR = CF::PR, PC = CF::PC, MR = CF::MR, MC = CF::MC, SC = CF::SC;
    const int N = p.N, S = p.S;
    const int gp = gl / PC, gq = gl - (gl / PC) * PC;
    float2 A[MR][MC], B[MR][SC];
#pragma unroll
    for (int v = 0; v < MC; ++v)
#pragma unroll
      for (int u = CF::umin(v); u < MR; ++u) {
        const int i = PR * u + gp, l = PC * v + gq;
        float2 x = make_float2(i == l ? 1.f : 0.f, 0.f);  // identity padding beyond N
        if (i < N && l < N) {
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
    float gam[SC];
    const int inf = chol_solve_group<CF>(N, S, A, B, sh, gl, bar_id, gam);
#pragma unroll
    for (int u = 0; u < MR; ++u)
#pragma unroll
      for (int kv = 0; kv < SC; ++kv) {
        const int i = PR * u + gp, k = PC * kv + gq;
        if (i < N && k < S) wsm[i * SMAX + k] = B[u][kv];
      }
    return inf;
  }
};

template <int NN, int LANES>
struct SmallSolverPolicy {
  static constexpr int G = LANES;
  static constexpr int kMaxThreads = 128, kMinBlocks = 5;  // registers <= 102: 5 CTAs (20 warps) per SM
  static constexpr bool kWInShared = true;                 // w_k aliases the L/U scratch after the solve
  static constexpr int kN = NN;
  using Shared = SmallShared<NN>;
  template <int C, int SMAX>
  __device__ static __forceinline__ int solve_bin(const KParams& p, const float2* blk, int W, int pr, float dlt,
                                                  const float2* __restrict__ steer, Shared& sh, int gl, int bar_id,
                                                  float2* wsm) {
    const int S = p.S;
    const int i = gl < NN ? gl : 0;
    float2 A[NN], Y[NN];
#pragma unroll
    for (int l = 0; l < NN; ++l) {
      float2 x = rhat_from_blocks(blk, C, W, pr, i, l);
      if (l == i) x = make_float2(x.x + dlt, 0.f);
      A[l] = x;
    }
    float g;
    const int inf = small_chol_solve<NN, LANES>(S, A, steer, Y, sh, gl, &g);
    if (gl < S) {
#pragma unroll
      for (int m = 0; m < NN; ++m) wsm[m * SMAX + gl] = Y[m];
    }
    return inf;
  }
};

// REMOTE: Y stores go through st_y (multicast / peer copies); the plain instantiation
// compiles to ordinary stores only.
template <int C, int SMAX, class SP, bool REMOTE>
__global__ void __launch_bounds__(SP::kMaxThreads, SP::kMinBlocks)
    fused_kernel(KParams p, const float2* __restrict__ cube, const float2* __restrict__ steer,
                 float2* __restrict__ out, int32_t* __restrict__ info, int P) {
  constexpr int G = SP::G;
  static_assert(!SP::kWInShared || sizeof(typename SP::Shared) >= (size_t)SP::kN * SMAX * 8, "w alias too small");
  extern __shared__ __align__(128) unsigned char smem[];
  const int run = blockIdx.x, b = blockIdx.y, n = blockIdx.z;
  const int T = p.T, K = p.K, N = p.N, S = p.S;
  const int ngroups = blockDim.x / G;
  const int dl0 = run * P;
  const int Prun = min(P, p.dop_count - dl0);
  const int d0 = p.dop_begin + dl0;
  const int W = Prun + T - 1;
  const FusedLayout lay = fused_layout(C, T, K, P, SP::kWInShared ? 0 : N, SMAX, ngroups,
                                       sizeof(typename SP::Shared));

  float2* xs = reinterpret_cast<float2*>(smem);
  float2* blk = reinterpret_cast<float2*>(smem + lay.off_blk);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + lay.off_bar);
  float* delta_s = reinterpret_cast<float*>(smem + lay.off_bar + 16);
  const int rs = tile_rs(K), bs = tile_bs(C, K);

  const int tid = threadIdx.x;
  const int grp = tid / G, gl = tid - grp * G;
  typename SP::Shared& sh = reinterpret_cast<typename SP::Shared*>(smem + lay.off_sh)[grp];
  // w_k as [N][SMAX]: its own region, or aliased onto this segment's solver scratch
  float2* wsm = SP::kWInShared ? reinterpret_cast<float2*>(&sh)
                               : reinterpret_cast<float2*>(smem + lay.off_w) + (size_t)grp * N * SMAX;
  const int bar_id = 1 + grp;

  STAPK_PROF_T(pt0);
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  for (int idx = gl; idx < N * SMAX; idx += G) wsm[idx] = make_float2(0.f, 0.f);  // zero padding columns
  __syncthreads();
  // 1-2. whole window resident (one chunk, KC = K) + lag-block HERK -> blk
  {
    CovLayout cl;
    cl.KC = K;
    cl.nchunks = 1;
    cl.nbuf = 1;
    cl.tile_bytes = lay.off_blk;
    cta_lag_blocks<C>(p, cube, n, b, d0, W, cl, smem, bar, blk);
  }
  if (tid < Prun) delta_s[tid] = delta_from_blocks(blk, C, T, N, p.lam, tid);
  __syncthreads();
  STAPK_PROF_T(pt1);
  if (tid == 0) STAPK_PROF_ADD(0, pt1 - pt0);

  // 4. bins round-robin over the solver segments (trip count uniform per warp)
  constexpr int GPW = G < 32 ? 32 / G : 1;
  const int wg0 = (grp / GPW) * GPW;
  for (int base = wg0; base < Prun; base += ngroups) {
    const int pr_raw = base + (grp - wg0);
    const bool valid = pr_raw < Prun;
    const int pr = valid ? pr_raw : Prun - 1;
    STAPK_PROF_T(ps0);
#if defined(STAPK_SKIP) && STAPK_SKIP >= 2  // dev builds only: phase-cost experiments
    const int inf = 0;
#else
    const int inf = SP::template solve_bin<C, SMAX>(p, blk, W, pr, delta_s[pr], steer, sh, gl, bar_id, wsm);
#endif
    chol_sync<G>(bar_id);
    STAPK_PROF_T(ps1);
    if (gl == 0) STAPK_PROF_ADD(1, ps1 - ps0);

    const int dl = dl0 + pr;
#if defined(STAPK_SKIP) && STAPK_SKIP >= 1
    if (valid && gl == 0) info[((long long)n * p.dop_count + dl) * p.B + b] = inf;
    if (false) {
#else
    if (valid) {
#endif
      if (gl == 0) info[((long long)n * p.dop_count + dl) * p.B + b] = inf;
      float2* yb = out + (((long long)n * p.dop_count + dl) * S) * p.R + (long long)b * K;
      const float2* xw = xs + pr * bs;
      // two range cells per lane per pass (j, j + G) share every weight load
      for (int j = gl; j < K; j += 2 * G) {
        const int j2 = j + G;
        const bool two = j2 < K;
        float2 acc0[SMAX], acc1[SMAX];
#pragma unroll
        for (int k = 0; k < SMAX; ++k) acc0[k] = acc1[k] = make_float2(0.f, 0.f);
        int i = 0;
        for (int t = 0; t < T; ++t) {
          for (int c = 0; c < C; ++c, ++i) {
            const float2* zr = xw + t * bs + c * rs;
            const float2 z0 = zr[j];
            const float2 z1 = two ? zr[j2] : make_float2(0.f, 0.f);
            const float4* wv = reinterpret_cast<const float4*>(wsm + i * SMAX);
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
        if constexpr (REMOTE) {
#pragma unroll
          for (int k = 0; k < SMAX; ++k)
            if (k < S) {
              st_y(yb + (long long)k * p.R + j, acc0[k], p);
              if (two) st_y(yb + (long long)k * p.R + j2, acc1[k], p);
            }
        } else {
#pragma unroll
          for (int k = 0; k < SMAX; ++k)
            if (k < S) {
              yb[(long long)k * p.R + j] = acc0[k];
              if (two) yb[(long long)k * p.R + j2] = acc1[k];
            }
        }
      }
    }
    chol_sync<G>(bar_id);
    STAPK_PROF_T(ps2);
    if (gl == 0) STAPK_PROF_ADD(2, ps2 - ps1);
  }
  STAPK_PROF_T(pt2);
  if (tid == 0) STAPK_PROF_ADD(3, pt2 - pt0);
}

// ---- host-side selection / launch ------------------------------------------
// (C, SMAX, N, solver) instantiations: the BASELINE.json shapes.
using FusedSolverTiny = SmallSolverPolicy<4, 16>;
using FusedSolverSmall = SmallSolverPolicy<12, 16>;
using FusedSolverMedium = CholSolverPolicy<CholCfg<4, 8, 8, 4, 2, false, 2>>;
#define STAPK_FUSED_CFGS(X)             \
  X(2, 4, 4, FusedSolverTiny)           \
  X(4, 16, 12, FusedSolverSmall)        \
  X(6, 16, 30, FusedSolverMedium)

inline int fused_smax(int S) { return S <= 2 ? 2 : S <= 4 ? 4 : S <= 8 ? 8 : S <= 16 ? 16 : 32; }

// Pick (P, threads) for the fused kernel; false -> use the staged path.
inline bool fused_configure(const KParams& kp, FusedCfg* f) {
  memset(f, 0, sizeof *f);
  const int SMAX = fused_smax(kp.S);
  int G = 0, maxT = 0, wN = 0;
  size_t shb = 0;
#define X(CC, SM, NN, SPT)                                       \
  if (kp.C == CC && SMAX == SM && kp.N == NN && kp.S <= 16) {    \
    G = SPT::G;                                                  \
    maxT = SPT::kMaxThreads;                                     \
    wN = SPT::kWInShared ? 0 : NN;                               \
    shb = sizeof(typename SPT::Shared);                          \
  }
  STAPK_FUSED_CFGS(X)
#undef X
  if (!G) return false;
  // the kernel's real register count (for the occupancy estimate)
  int regs = 128;
  {
    cudaFuncAttributes fa;
    bool got = false;
#define X(CC, SM, NN, SPT)                                                            \
    if (!got && kp.C == CC && SMAX == SM && kp.N == NN)                                \
      got = cudaFuncGetAttributes(&fa, fused_kernel<CC, SM, SPT, false>) == cudaSuccess;
    STAPK_FUSED_CFGS(X)
#undef X
    if (got) regs = fa.numRegs;
    cudaGetLastError();
  }
  const int regs_alloc = (regs + 7) & ~7;
  const size_t cap = 227 * 1024;
  int bestP = 0, bestT = 0;
  size_t bestS = 0;
  double bestScore = -1.0;
  for (int threads = 128; threads <= maxT; threads += 128) {
    if (threads % G) continue;
    const int ng = threads / G;
    for (int P = 1; P <= kp.dop_count && P <= 64; ++P) {
      if (cov_tpb(kp.C) * cov_blocks(kp.T, P + kp.T - 1) > threads) break;
      const FusedLayout L = fused_layout(kp.C, kp.T, kp.K, P, wN, SMAX, ng, shb);
      if (L.total > cap) break;
      int cta_per_sm = (int)((228 * 1024) / (L.total + 1024));    // shared memory
      const int by_regs = 65536 / (regs_alloc * threads);         // register file
      if (by_regs < cta_per_sm) cta_per_sm = by_regs;
      if (2048 / threads < cta_per_sm) cta_per_sm = 2048 / threads;
      if (cta_per_sm < 1) break;
      const int warps = cta_per_sm * threads / 32;
      // solver segments work in rounds of ng bins: the last round of a run of P
      // bins is P mod ng busy, so weight by the round balance
      const double balance = (double)P / ((double)((P + ng - 1) / ng) * ng);
      // prefer more busy resident warps and CTAs (independent phases overlap),
      // then less covariance work per bin (larger P)
      const double score = (warps > 32 ? 32 : warps) * balance * 1000.0 + cta_per_sm * 10.0 + P * 0.01;
      if (score > bestScore) {
        bestScore = score;
        bestP = P;
        bestT = threads;
        bestS = L.total;
      }
    }
  }
  // the fused kernel only pays with enough busy resident warps to overlap its
  // phases (>= 12 per SM) and when the lag blocks keep >= 1/3 of the threads busy
  if (bestP == 0 || bestScore < 12000.0 || 3 * cov_tpb(kp.C) * cov_blocks(kp.T, bestP + kp.T - 1) < bestT)
    return false;
  f->C = kp.C;
  f->SMAX = SMAX;
  f->N = kp.N;
  f->G = G;
  f->P = bestP;
  f->threads = bestT;
  f->runs = (kp.dop_count + bestP - 1) / bestP;
  f->smem = bestS;
  snprintf(f->name, sizeof f->name, "C=%d,SMAX=%d,N=%d,G=%d,P=%d,threads=%d,smem=%zu", kp.C, SMAX, kp.N, G, bestP,
           bestT, bestS);
  return true;
}

inline void fused_set_attr(const FusedCfg& f) {
#define X(CC, SM, NN, SPT)                                                                                         \
  if (f.C == CC && f.SMAX == SM && f.N == NN) {                                                                    \
    cudaFuncSetAttribute(fused_kernel<CC, SM, SPT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f.smem); \
    cudaFuncSetAttribute(fused_kernel<CC, SM, SPT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f.smem);  \
  }
  STAPK_FUSED_CFGS(X)
#undef X
}

inline void fused_launch(const FusedCfg& f, const KParams& kp, const float2* cube, const float2* steer,
                         float2* out, int32_t* info, cudaStream_t st) {
  dim3 grid(f.runs, kp.B, kp.batch);
#define X(CC, SM, NN, SPT)                                                                       \
  if (f.C == CC && f.SMAX == SM && f.N == NN) {                                                  \
    if (kp.y_mc | kp.y_np)                                                                       \
      fused_kernel<CC, SM, SPT, true><<<grid, f.threads, f.smem, st>>>(kp, cube, steer, out, info, f.P); \
    else                                                                                         \
      fused_kernel<CC, SM, SPT, false><<<grid, f.threads, f.smem, st>>>(kp, cube, steer, out, info, f.P); \
  }
  STAPK_FUSED_CFGS(X)
#undef X
}

}  // namespace stapk

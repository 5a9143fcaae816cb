// cholsm.cuh -- K2 (N > 16), shared-memory-resident blocked solver: batched Hermitian
// Cholesky + forward/back solves -> MVDR weights, one matrix per 128-thread CTA at a time.
//
// Method (include/stap.h; readings c-9, c-10, c-11, r-5): R = L L^H; y_k = L^-1 s_k;
// gamma_k = ||y_k||^2; w_k = L^-H y_k / gamma_k; info as in chol.cuh.  The same
// square-root-free arithmetic as chol.cuh: the factor is kept raw (a_j = L[:,j] sqrt(p_j)),
// A[i][l] -= a_i conj(a_l) / p_j, B[i][k] -= a_i yraw_j[k] / p_j, gamma_k = sum |yraw|^2 / p,
// v_i = (yraw_i - sum_{m>i} conj(a_m^(i)) v_m) / p_i -- one rcp per pivot.
//
// Why a second solver design: the register-resident one (chol.cuh) keeps ~20 KB of state per
// matrix in registers, so only 8 matrices fit an SM and its 112 dependent per-step chains
// (barrier, shared round trip, rcp) are exposed.  Here the matrix lives in shared memory
// (~40 KB with the right-hand sides at N = 56), five CTAs per SM, and the work is blocked by
// panels of 8 columns (right-looking):
//   P  one warp factors the panel (8 columns, rows >= j0) in registers with shuffles, and
//      forward-solves the panel's 8 right-hand-side rows (lane = k);
//   T  all 128 threads apply the rank-8 update to the trailing matrix and right-hand sides in
//      4x2 register tiles (raw panel rows x scaled panel rows): 16-byte shared loads, FFMA2;
// then the back solve by panels from the bottom: one warp solves the 8 x 8 triangle for its
// right-hand sides, all threads apply the rank-8 update to the rows above.  Two __syncthreads
// per panel instead of a barrier per column.
#pragma once
#include "common.cuh"

namespace stapk {

__device__ __forceinline__ float rcp_approx_sm(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

template <int NP_, int SP_>
struct CholSmCfg {
  static constexpr int NP = NP_;      // N padded to a multiple of 8 (identity padding), <= 64
  static constexpr int SP = SP_;      // S padded: 16 or 32 (zero right-hand sides)
  static constexpr int NB = NP / 8;   // panels
  static constexpr int LDA = NP + 2;  // float2 row stride of A (16-byte rows, 4 banks apart)
  static constexpr int LDB = SP + 2;  // of B
  static constexpr int LDP = 9;       // of the scaled panel Ps (8 used; odd: conflict-free 8-byte reads)
  static constexpr int kThreads = 128;
  static_assert(NP % 8 == 0 && NP <= 64 && NP >= 8, "panels of 8");
  static_assert(SP == 16 || SP == 32, "right-hand sides per lane of the panel warp");
  // shared memory (float2 counts, then floats)
  static constexpr size_t kA = (size_t)NP * LDA, kB = (size_t)NP * LDB, kP = (size_t)NP * LDP, kY = 8 * (size_t)SP;
  static constexpr size_t kBytes = (kA + kB + kP + kY) * 8 + (2 * NP + SP + 8) * 4;
};

template <class CF, int kMinBlocks>
__global__ void __launch_bounds__(128, kMinBlocks)
    cholsm_kernel(int N, int S, long long units, const float2* __restrict__ cov, const float2* __restrict__ steer,
                  float2* __restrict__ wout, float* __restrict__ gout, int32_t* __restrict__ info) {
  constexpr int NP = CF::NP, SP = CF::SP, NB = CF::NB, LDA = CF::LDA, LDB = CF::LDB, LDP = CF::LDP;
  extern __shared__ __align__(128) unsigned char smem[];
  float2* A = reinterpret_cast<float2*>(smem);  // [NP][LDA]: the matrix, then the raw factor
  float2* Bm = A + CF::kA;                        // [NP][LDB]: right-hand sides -> yraw -> v
  float2* Ps = Bm + CF::kB;                       // [NP][LDP]: the current panel, scaled by 1/p
  float2* Ys = Ps + CF::kP;                       // [8][SP]: the panel's yraw rows, scaled by 1/p
  float* piv = reinterpret_cast<float*>(Ys + CF::kY);  // [NP] pivots
  float* rpv = piv + NP;                               // [NP] 1/pivot
  float* gam = rpv + NP;                               // [SP]
  int* flag = reinterpret_cast<int*>(gam + SP);        // [8] info scratch
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  for (long long u = blockIdx.x; u < units; u += gridDim.x) {
    // ---- load: lower triangle of R (identity padding beyond N), zero above; the steering set
    // (all of a thread's loads are issued before its first store: one memory latency per matrix)
    const float2* Rg = cov + u * N * N;
    constexpr int kPairs = NP * NP / 2, kPer = (kPairs + CF::kThreads - 1) / CF::kThreads;
    float4 ld[kPer];
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int idx = tid + t * CF::kThreads;  // pair (i, 2*lp), (i, 2*lp+1)
      const int i = idx / (NP / 2), l = 2 * (idx - i * (NP / 2));
      float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
      if (idx < kPairs && l <= i) {
        if (i < N && l + 1 < N && (N & 1) == 0) {
          x = __ldg(reinterpret_cast<const float4*>(Rg + i * N + l));
        } else {
          const float2 x0 = i < N && l < N ? __ldg(Rg + i * N + l) : make_float2(i == l ? 1.f : 0.f, 0.f);
          const float2 x1 = i < N && l + 1 < N ? __ldg(Rg + i * N + l + 1) : make_float2(i == l + 1 ? 1.f : 0.f, 0.f);
          x = make_float4(x0.x, x0.y, x1.x, x1.y);
        }
        if (l + 1 > i) x.z = x.w = 0.f;  // above the diagonal
      }
      ld[t] = x;
    }
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int idx = tid + t * CF::kThreads;
      const int i = idx / (NP / 2), l = 2 * (idx - i * (NP / 2));
      if (idx < kPairs) *reinterpret_cast<float4*>(A + i * LDA + l) = ld[t];
    }
    for (int idx = tid; idx < NP * SP; idx += CF::kThreads) {
      const int i = idx / SP, k = idx - i * SP;
      Bm[i * LDB + k] = (i < N && k < S) ? __ldg(steer + k * N + i) : make_float2(0.f, 0.f);
    }
    __syncthreads();

    // ---- Cholesky + forward solve, by panels of 8 columns
#pragma unroll 1
    for (int J = 0; J < NB; ++J) {
      const int j0 = 8 * J;
      if (warp == 0) {
        // P: rows j0 + lane (pa) and j0 + 32 + lane (pb) of the panel; lane k < SP: rows j0..j0+7 of B
        const int ra = j0 + lane, rb = j0 + 32 + lane;
        float2 pa[8], pb[8], bj[8];
#pragma unroll
        for (int c = 0; c < 8; c += 2) {
          if (ra < NP) {
            const float4 v = *reinterpret_cast<const float4*>(A + ra * LDA + j0 + c);
            pa[c] = make_float2(v.x, v.y);
            pa[c + 1] = make_float2(v.z, v.w);
          } else {
            pa[c] = pa[c + 1] = make_float2(0.f, 0.f);
          }
          if (rb < NP) {
            const float4 v = *reinterpret_cast<const float4*>(A + rb * LDA + j0 + c);
            pb[c] = make_float2(v.x, v.y);
            pb[c + 1] = make_float2(v.z, v.w);
          } else {
            pb[c] = pb[c + 1] = make_float2(0.f, 0.f);
          }
        }
#pragma unroll
        for (int a = 0; a < 8; ++a) bj[a] = lane < SP ? Bm[(j0 + a) * LDB + lane] : make_float2(0.f, 0.f);
        float r2s[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const float pv = __shfl_sync(0xffffffffu, pa[jj].x, jj);  // A[j][j], j = j0 + jj
          const float r2 = rcp_approx_sm(pv);
          r2s[jj] = r2;
          if (lane == 0) {
            piv[j0 + jj] = pv;
            rpv[j0 + jj] = r2;
          }
#pragma unroll
          for (int c = jj + 1; c < 8; ++c) {
            // a_l for l = j0 + c (row l of column j, lane c), scaled by 1/p_j
            const float2 lc = make_float2(__shfl_sync(0xffffffffu, pa[jj].x, c) * r2,
                                          __shfl_sync(0xffffffffu, pa[jj].y, c) * r2);
            cmsub_conjb2(pa[c], pa[jj], lc);  // rows above the diagonal become garbage, never read
            cmsub_conjb2(pb[c], pb[jj], lc);
            cmsub2(bj[c], lc, bj[jj]);        // B[l][k] -= (a_l / p_j) yraw_j[k]
          }
        }
        // publish: raw panel -> A, scaled panel -> Ps, the panel's yraw -> B and scaled -> Ys
#pragma unroll
        for (int c = 0; c < 8; c += 2) {
          if (ra < NP)
            *reinterpret_cast<float4*>(A + ra * LDA + j0 + c) = make_float4(pa[c].x, pa[c].y, pa[c + 1].x, pa[c + 1].y);
          if (rb < NP)
            *reinterpret_cast<float4*>(A + rb * LDA + j0 + c) = make_float4(pb[c].x, pb[c].y, pb[c + 1].x, pb[c + 1].y);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (ra < NP) Ps[ra * LDP + c] = make_float2(pa[c].x * r2s[c], pa[c].y * r2s[c]);
          if (rb < NP) Ps[rb * LDP + c] = make_float2(pb[c].x * r2s[c], pb[c].y * r2s[c]);
        }
        if (lane < SP) {
#pragma unroll
          for (int a = 0; a < 8; ++a) {
            Bm[(j0 + a) * LDB + lane] = bj[a];
            Ys[a * SP + lane] = make_float2(bj[a].x * r2s[a], bj[a].y * r2s[a]);
          }
        }
      }
      __syncthreads();
      // T: rank-8 update of rows/cols >= t0 (A lower triangle in 4x2 tiles) and of B rows >= t0
      const int t0 = j0 + 8;
      const int MA = (NP - t0) / 4;   // row tiles
      const int nA = MA * MA + MA;    // lower-triangle 4x2 tiles: row tile a has 2a + 2
      const int nBt = MA * (SP / 2);  // B tiles
      for (int idx = tid; idx < nA + nBt; idx += CF::kThreads) {
        int a, b;
        const bool isA = idx < nA;
        if (isA) {
          a = (int)((sqrtf(4.f * (float)idx + 1.f) - 1.f) * 0.5f);
          while ((a + 1) * (a + 2) <= idx) ++a;  // guard the float estimate
          while (a * (a + 1) > idx) --a;
          b = idx - a * (a + 1);
        } else {
          const int q = idx - nA;
          a = q / (SP / 2);
          b = q - a * (SP / 2);
        }
        const int i0 = t0 + 4 * a;
        float2* dst = isA ? A + i0 * LDA + t0 + 2 * b : Bm + i0 * LDB + 2 * b;
        const int ld = isA ? LDA : LDB;
        float2 acc[4][2];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const float4 v = *reinterpret_cast<const float4*>(dst + r * ld);
          acc[r][0] = make_float2(v.x, v.y);
          acc[r][1] = make_float2(v.z, v.w);
        }
#pragma unroll
        for (int c = 0; c < 8; c += 2) {
          float2 pr[4][2], sc[2][2];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const float4 v = *reinterpret_cast<const float4*>(A + (i0 + r) * LDA + j0 + c);
            pr[r][0] = make_float2(v.x, v.y);
            pr[r][1] = make_float2(v.z, v.w);
          }
          if (isA) {
            const int l0 = t0 + 2 * b;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              sc[q][0] = Ps[(l0 + q) * LDP + c];
              sc[q][1] = Ps[(l0 + q) * LDP + c + 1];
            }
#pragma unroll
            for (int cc = 0; cc < 2; ++cc)
#pragma unroll
              for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int q = 0; q < 2; ++q) cmsub_conjb2(acc[r][q], pr[r][cc], sc[q][cc]);
          } else {
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
              const float4 v = *reinterpret_cast<const float4*>(Ys + (c + cc) * SP + 2 * b);
              sc[0][cc] = make_float2(v.x, v.y);
              sc[1][cc] = make_float2(v.z, v.w);
            }
#pragma unroll
            for (int cc = 0; cc < 2; ++cc)
#pragma unroll
              for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int q = 0; q < 2; ++q) cmsub2(acc[r][q], pr[r][cc], sc[q][cc]);
          }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
          *reinterpret_cast<float4*>(dst + r * ld) = make_float4(acc[r][0].x, acc[r][0].y, acc[r][1].x, acc[r][1].y);
      }
      __syncthreads();
    }

    // ---- gamma_k = sum_i |yraw_i[k]|^2 / p_i (ascending i); info from the pivots
    if (tid < SP) {
      float g = 0.f;
      for (int i = 0; i < N; ++i) {
        const float2 y = Bm[i * LDB + tid];
        g = fmaf(fmaf(y.x, y.x, y.y * y.y), rpv[i], g);
      }
      gam[tid] = g;
    }
    if (warp == 1) {
      int fail = 0;
#pragma unroll
      for (int j0 = 0; j0 < NP; j0 += 32) {
        const int j = j0 + lane;
        const unsigned m = __ballot_sync(0xffffffffu, j < N && !finite_pos(piv[j < N ? j : 0]));
        if (!fail && m) fail = j0 + __ffs(m);
      }
      if (lane == 0) flag[0] = fail;
    }

    // ---- back solve by panels from the bottom
#pragma unroll 1
    for (int J = NB - 1; J >= 0; --J) {
      const int j0 = 8 * J;
      if (warp == 0 && lane < SP) {
        // Pb: the 8 x 8 triangle for right-hand side k = lane
        float2 t[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) t[a] = Bm[(j0 + a) * LDB + lane];
#pragma unroll
        for (int a = 7; a >= 0; --a) {
          const float ra = rpv[j0 + a];
          t[a] = make_float2(t[a].x * ra, t[a].y * ra);  // v_{j0+a}
#pragma unroll
          for (int c = 0; c < a; ++c) cmsub_conja2(t[c], A[(j0 + a) * LDA + j0 + c], t[a]);
        }
#pragma unroll
        for (int a = 0; a < 8; ++a) Bm[(j0 + a) * LDB + lane] = t[a];
      }
      __syncthreads();
      // Tb: rows m < j0 of B: t_m -= sum_a conj(a_{j0+a}^(m)) v_{j0+a}, tiles of 4 rows x 2 k
      const int nT = (j0 / 4) * (SP / 2);
      for (int idx = tid; idx < nT; idx += CF::kThreads) {
        const int a4 = idx / (SP / 2), b = idx - a4 * (SP / 2);
        const int m0 = 4 * a4;
        float2* dst = Bm + m0 * LDB + 2 * b;
        float2 acc[4][2];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const float4 v = *reinterpret_cast<const float4*>(dst + r * LDB);
          acc[r][0] = make_float2(v.x, v.y);
          acc[r][1] = make_float2(v.z, v.w);
        }
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          const float4 l01 = *reinterpret_cast<const float4*>(A + (j0 + a) * LDA + m0);
          const float4 l23 = *reinterpret_cast<const float4*>(A + (j0 + a) * LDA + m0 + 2);
          const float4 vv = *reinterpret_cast<const float4*>(Bm + (j0 + a) * LDB + 2 * b);
          const float2 lr[4] = {make_float2(l01.x, l01.y), make_float2(l01.z, l01.w), make_float2(l23.x, l23.y),
                                make_float2(l23.z, l23.w)};
          const float2 v[2] = {make_float2(vv.x, vv.y), make_float2(vv.z, vv.w)};
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int q = 0; q < 2; ++q) cmsub_conja2(acc[r][q], lr[r], v[q]);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
          *reinterpret_cast<float4*>(dst + r * LDB) = make_float4(acc[r][0].x, acc[r][0].y, acc[r][1].x, acc[r][1].y);
      }
      __syncthreads();
    }

    // ---- normalise, zero failed k / unit, store W [S][N], gamma, info
    const int fail = flag[0];
    for (int idx = tid; idx < S * N; idx += CF::kThreads) {
      const int k = idx / N, i = idx - k * N;
      const float g = gam[k];
      const bool ok = finite_pos(g) && !fail;
      const float ig = ok ? 1.0f / g : 0.f;
      const float2 v = Bm[i * LDB + k];
      wout[u * S * N + idx] = ok ? make_float2(v.x * ig, v.y * ig) : make_float2(0.f, 0.f);
    }
    if (tid < S && gout) gout[u * S + tid] = (fail || !finite_pos(gam[tid])) ? 0.f : gam[tid];
    if (warp == 2) {
      int bad = 0;
      for (int k0 = 0; k0 < S; k0 += 32) {
        const int k = k0 + lane;
        const unsigned m = __ballot_sync(0xffffffffu, k < S && !finite_pos(gam[k < S ? k : 0]));
        if (!bad && m) bad = k0 + __ffs(m);
      }
      if (lane == 0) info[u] = fail ? fail : (bad ? -bad : 0);
    }
    __syncthreads();  // every thread is done with the buffers before the next matrix loads
  }
}

// ---- host-side selection ---------------------------------------------------
#define STAPK_CHOLSM_CFGS(X)        \
  X(0, (CholSmCfg<24, 16>), 8)      \
  X(1, (CholSmCfg<32, 16>), 8)      \
  X(2, (CholSmCfg<40, 16>), 6)      \
  X(3, (CholSmCfg<48, 16>), 6)      \
  X(4, (CholSmCfg<56, 16>), 5)      \
  X(5, (CholSmCfg<64, 16>), 4)      \
  X(6, (CholSmCfg<24, 32>), 8)      \
  X(7, (CholSmCfg<32, 32>), 6)      \
  X(8, (CholSmCfg<40, 32>), 5)      \
  X(9, (CholSmCfg<48, 32>), 4)      \
  X(10, (CholSmCfg<56, 32>), 4)     \
  X(11, (CholSmCfg<64, 32>), 3)

struct CholSmSel {
  int id = -1;
  size_t smem = 0;
  int min_blocks = 0;
};

#define STAPK_UNPAREN_SM_I(...) __VA_ARGS__
#define STAPK_UNPAREN_SM STAPK_UNPAREN_SM_I

inline bool cholsm_select(int N, int S, CholSmSel* sel) {
  if (N < 17 || N > 64 || S < 1 || S > 32) return false;
  const int np = (N + 7) / 8 * 8;
  const int id = (np / 8 - 3) + (S > 16 ? 6 : 0);
  switch (id) {
#define X(I, CFT, MB)                           \
  case I: {                                     \
    using CF_ = STAPK_UNPAREN_SM CFT;           \
    sel->id = I;                                \
    sel->smem = CF_::kBytes;                    \
    sel->min_blocks = MB;                       \
    break;                                      \
  }
    STAPK_CHOLSM_CFGS(X)
#undef X
    default: return false;
  }
  return true;
}

inline cudaError_t cholsm_set_attr(const CholSmSel& s) {
  switch (s.id) {
#define X(I, CFT, MB) \
  case I: return cudaFuncSetAttribute(cholsm_kernel<STAPK_UNPAREN_SM CFT, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s.smem);
    STAPK_CHOLSM_CFGS(X)
#undef X
  }
  return cudaErrorInvalidValue;
}

inline void cholsm_launch(const CholSmSel& s, int grid, cudaStream_t st, int N, int S, long long units,
                          const float2* cov, const float2* steer, float2* w, float* g, int32_t* info) {
  switch (s.id) {
#define X(I, CFT, MB) \
  case I: cholsm_kernel<STAPK_UNPAREN_SM CFT, MB><<<grid, 128, s.smem, st>>>(N, S, units, cov, steer, w, g, info); break;
    STAPK_CHOLSM_CFGS(X)
#undef X
  }
}

}  // namespace stapk

// solve.cuh -- K2: batched Hermitian Cholesky + forward/back solves -> MVDR weights.
//
// Method (include/stap.h; readings c-9, c-10, c-11): R = L L^H with L lower and a
// real positive diagonal; y_k = L^-1 s_k; gamma_k = ||y_k||^2; v_k = L^-H y_k
// (= R^-1 s_k); w_k = v_k / gamma_k.  A non-positive / non-finite pivot j sets
// info = j+1 and zeroes the unit's weights; a bad gamma_k sets info = -(k+1)
// for the smallest such k and zeroes w_k.
//
// B200 design: one lane GROUP of PR x PC lanes per matrix (8 lanes for N <= 8
// ... 64 lanes = 2 warps for N <= 64), the matrix REGISTER-resident in a 2-D
// block-cyclic layout: element (i, l) of the lower triangle lives in lane
// (i mod PR, l mod PC), register [i / PR][l / PC]; right-hand side element
// (i, k) in lane (i mod PR, k mod PC), register [i / PR][k / PC].
//   Cholesky + forward solve, right-looking: step j scales column j (its owners
//   publish it in shared memory), finalises y_j (row-j owners publish it), and
//   every lane applies the rank-1 update A[i][l] -= L[i][j] conj(L[l][j]) and
//   B[i][k] -= L[i][j] y_j[k] to the elements it owns -- all independent FMAs.
//   Back solve, row by row from the bottom: row i of L and v_i are published,
//   every lane updates its rows above.
// Register indices are compile-time (outer loops over register blocks are
// unrolled, the inner position inside a block is a runtime loop), so nothing
// spills to local memory.  Two group barriers per step; a failed pivot does not
// break the loop (groups sharing a warp keep a uniform control flow).
#pragma once
#include <cstdlib>

#include "common.cuh"

namespace stapk {

template <int PR_, int PC_, int MR_, int MC_, int SC_>
struct SolveCfg {
  static constexpr int PR = PR_, PC = PC_, MR = MR_, MC = MC_, SC = SC_;
  static constexpr int G = PR * PC;        // lanes per matrix
  static constexpr int NMAX = (PR * MR < PC * MC) ? PR * MR : PC * MC;
  static constexpr int SMAXC = PC * SC;    // right-hand sides per matrix (capacity)
  // smallest register row-block u that can hold a lower-triangle element of register column-block v
  __host__ __device__ static constexpr int umin(int v) { return (PC * v - PR + 1) <= 0 ? 0 : (PC * v - PR + 1 + PR - 1) / PR; }
};

// Per-group shared scratch (floats / float2), sized for the config.
template <class CF>
struct SolveShared {
  // double-buffered by the parity of the step, so that groups of more than one warp
  // (bar.sync) need one group barrier per step (kOneBarrier below)
  float2 col[2][CF::PR * CF::MR];  // raw column j of the factor (rows), pivot at [j]
  float2 row[2][CF::PC * CF::MC];  // row i of L (columns), back solve
  float2 yb[2][CF::SMAXC];         // raw y_j (forward) / v_i (backward)
  float rdiag[CF::PR * CF::MR];  // 1 / L[j][j]
  float gpart[CF::PR][CF::SMAXC];
  float gam[CF::SMAXC];
  float xj;
  int fail;
};

template <int G>
__device__ __forceinline__ void group_sync(int bar_id) {
  if constexpr (G <= 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(G) : "memory");
  }
}

// Solve one matrix per group.  A must hold the lower triangle of R (entries with
// row < N, col <= row; others are ignored), B the steering rows B[i][k] = s_k[i].
// On return B holds w_k[i] (0 for failed k / failed unit) and the function
// returns info (identical on all lanes of the group).  gam_out (lane-local,
// per register column kv) receives gamma_k for the lane's k's.
template <class CF>
__device__ __forceinline__ int group_chol_solve(int N, int S, float2 (&A)[CF::MR][CF::MC], float2 (&B)[CF::MR][CF::SC],
                                                SolveShared<CF>& sh, int gl, int bar_id) {
  constexpr int PR = CF::PR, PC = CF::PC, MR = CF::MR, MC = CF::MC, SC = CF::SC, G = CF::G;
  const int p = gl / PC, q = gl - (gl / PC) * PC;
  int fail = 0;
  // Groups of more than one warp synchronise with bar.sync, whose cost dominates a step:
  // they publish pivot, column and y_j together into parity buffers (one barrier per step,
  // large solve 2.33 -> 2.23 ms).  Single-warp groups (__syncwarp) keep the two-barrier
  // step, which measured faster for them (medium solve 1.22 vs 1.32 ms).
  constexpr bool kOneBarrier = G > 32;

  // ---------------- Cholesky + forward solve (right-looking)
#pragma unroll
  for (int v = 0; v < MC; ++v) {
    for (int qq = 0; qq < PC; ++qq) {
      const int j = PC * v + qq;
      if (j >= N) break;  // uniform
      const int pj = j % PR, uj = j / PR, bp = kOneBarrier ? (j & 1) : 0;
      float r;
      if constexpr (kOneBarrier) {
        // (a) column-j owners publish the RAW column j (its diagonal entry is the pivot),
        // row-j owners the RAW y_j; consumers scale by r = 1/sqrt(pivot) themselves.
        // Parity buffers: a lane can only write buffer bp again (step j+2) after every
        // lane has passed step j+1's barrier, i.e. finished reading step j's.
        if (q == qq) {
#pragma unroll
          for (int u = CF::umin(v); u < MR; ++u) sh.col[bp][PR * u + p] = A[u][v];
        }
        if (p == pj) {
#pragma unroll
          for (int u = (PC * v) / PR; u <= (PC * v + PC - 1) / PR && u < MR; ++u)
            if (u == uj) {
#pragma unroll
              for (int kv = 0; kv < SC; ++kv) sh.yb[bp][PC * kv + q] = B[u][kv];
            }
        }
        group_sync<G>(bar_id);
        // (b) every lane: pivot, 1/sqrt; row-j owners finalise y_j
        float x = sh.col[bp][j].x;
        const bool ok = finite_pos(x);
        if (!ok && !fail) fail = j + 1;
        if (!ok) x = 1.0f;
        r = rsqrtf(x);  // one MUFU on the pivot chain
        if (gl == 0) sh.rdiag[j] = r;
        if (p == pj) {
#pragma unroll
          for (int u = (PC * v) / PR; u <= (PC * v + PC - 1) / PR && u < MR; ++u)
            if (u == uj) {
#pragma unroll
              for (int kv = 0; kv < SC; ++kv) {
                B[u][kv].x *= r;
                B[u][kv].y *= r;
              }
            }
        }
      } else {
        // (a) diag owner publishes the pivot
        if (p == pj && q == qq) {
          float x = 0.f;
#pragma unroll
          for (int u = (PC * v) / PR; u <= (PC * v + PC - 1) / PR && u < MR; ++u)
            if (u == uj) x = A[u][v].x;
          sh.xj = x;
        }
        group_sync<G>(bar_id);
        // (b) every lane: pivot, scale column j / finalise y_j
        float x = sh.xj;
        const bool ok = finite_pos(x);
        if (!ok && !fail) fail = j + 1;
        if (!ok) x = 1.0f;
        r = rsqrtf(x);  // one MUFU on the pivot chain
        if (gl == 0) sh.rdiag[j] = r;
        // column j is published RAW (consumers scale by r); the owners keep it raw
        if (q == qq) {
#pragma unroll
          for (int u = CF::umin(v); u < MR; ++u) sh.col[0][PR * u + p] = A[u][v];
        }
        if (p == pj) {
#pragma unroll
          for (int u = (PC * v) / PR; u <= (PC * v + PC - 1) / PR && u < MR; ++u) {
            if (u == uj) {
#pragma unroll
              for (int kv = 0; kv < SC; ++kv) {
                B[u][kv].x *= r;
                B[u][kv].y *= r;
                sh.yb[0][PC * kv + q] = B[u][kv];
              }
            }
          }
        }
        group_sync<G>(bar_id);
      }
      // (c) rank-1 update of the trailing matrix and of the right-hand sides
      float2 Li[MR], Ll[MC], yk[SC];
#pragma unroll
      for (int u = CF::umin(v); u < MR; ++u) {
        const float2 c = sh.col[bp][PR * u + p];
        Li[u] = make_float2(c.x * r, c.y * r);  // L[i][j]
      }
#pragma unroll
      for (int v2 = v; v2 < MC; ++v2) {
        const float2 c = sh.col[bp][PC * v2 + q];
        Ll[v2] = make_float2(c.x * r, c.y * r);  // L[l][j]
      }
#pragma unroll
      for (int kv = 0; kv < SC; ++kv) {
        const float2 c = sh.yb[bp][PC * kv + q];
        yk[kv] = kOneBarrier ? make_float2(c.x * r, c.y * r) : c;  // y_j[k]
      }
      // Only lower-triangle entries right of column j must change; the others a
      // lane holds (upper triangle, rows >= N) are never read as results, so
      // they are updated unconditionally (no per-element predicate).
      if (q > qq) {
#pragma unroll
        for (int u = CF::umin(v); u < MR; ++u) cmsub_conjb2(A[u][v], Li[u], Ll[v]);
      }
#pragma unroll
      for (int v2 = v + 1; v2 < MC; ++v2) {
#pragma unroll
        for (int u = CF::umin(v2); u < MR; ++u) cmsub_conjb2(A[u][v2], Li[u], Ll[v2]);
      }
#pragma unroll
      for (int u = CF::umin(v); u < MR; ++u) {
        if (PR * u + p > j) {  // finalised rows <= j keep y
#pragma unroll
          for (int kv = 0; kv < SC; ++kv) cmsub2(B[u][kv], Li[u], yk[kv]);
        }
      }
    }
  }
  if constexpr (kOneBarrier) group_sync<G>(bar_id);  // rdiag[N-1] was written after the last step's barrier
  // deferred column scaling: L[i][l] = raw[i][l] / sqrt(pivot_l) for every held entry
  // (diagonal and upper-triangle entries become garbage: the back solve never reads them)
#pragma unroll
  for (int v = 0; v < MC; ++v) {
    const float rl = sh.rdiag[(PC * v + q) < N ? PC * v + q : 0];
#pragma unroll
    for (int u = CF::umin(v); u < MR; ++u) {
      A[u][v].x *= rl;
      A[u][v].y *= rl;
    }
  }

  // ---------------- gamma_k = ||y_k||^2 (lane partials over its rows, then a fixed-order sum over p)
  float gl_part[SC];
#pragma unroll
  for (int kv = 0; kv < SC; ++kv) {
    float g = 0.f;
#pragma unroll
    for (int u = 0; u < MR; ++u) {
      if (PR * u + p < N) {
        g = fmaf(B[u][kv].x, B[u][kv].x, g);
        g = fmaf(B[u][kv].y, B[u][kv].y, g);
      }
    }
    gl_part[kv] = g;
    sh.gpart[p][PC * kv + q] = g;
  }
  group_sync<G>(bar_id);
  if (p == 0) {
#pragma unroll
    for (int kv = 0; kv < SC; ++kv) {
      float g = 0.f;
#pragma unroll
      for (int pp = 0; pp < PR; ++pp) g += sh.gpart[pp][PC * kv + q];
      sh.gam[PC * kv + q] = g;
    }
  }
  group_sync<G>(bar_id);
  (void)gl_part;

  // ---------------- back solve v = L^-H y (rows from the bottom)
#pragma unroll
  for (int ui = MR - 1; ui >= 0; --ui) {
    for (int pi = PR - 1; pi >= 0; --pi) {
      const int i = PR * ui + pi, bb = kOneBarrier ? (i & 1) : 0;  // parity buffers, as in the forward loop
      if (i >= N) continue;  // uniform
      if (p == pi) {
#pragma unroll
        for (int v = 0; v < MC; ++v)
          if (ui >= CF::umin(v)) sh.row[bb][PC * v + q] = A[ui][v];
        const float r = sh.rdiag[i];
#pragma unroll
        for (int kv = 0; kv < SC; ++kv) {
          B[ui][kv].x *= r;
          B[ui][kv].y *= r;
          sh.yb[bb][PC * kv + q] = B[ui][kv];
        }
      }
      group_sync<G>(bar_id);
      float2 vk[SC];
#pragma unroll
      for (int kv = 0; kv < SC; ++kv) vk[kv] = sh.yb[bb][PC * kv + q];
#pragma unroll
      for (int u = 0; u < ui; ++u) {  // rows m = PR*u + p < i
        const float2 lim = sh.row[bb][PR * u + p];
#pragma unroll
        for (int kv = 0; kv < SC; ++kv) cmsub_conja2(B[u][kv], lim, vk[kv]);
      }
      if (p < pi) {
        const float2 lim = sh.row[bb][PR * ui + p];
#pragma unroll
        for (int kv = 0; kv < SC; ++kv) cmsub_conja2(B[ui][kv], lim, vk[kv]);
      }
      if constexpr (!kOneBarrier) group_sync<G>(bar_id);
    }
  }
  if constexpr (kOneBarrier) group_sync<G>(bar_id);  // every lane is done reading the last row's buffers

  // ---------------- normalise: w_k = v_k / gamma_k; zero failed k or a failed unit
#pragma unroll
  for (int kv = 0; kv < SC; ++kv) {
    const int k = PC * kv + q;
    const float g = sh.gam[k];
    const bool gok = finite_pos(g) && !fail;
    const float ig = gok ? 1.0f / g : 0.f;
#pragma unroll
    for (int u = 0; u < MR; ++u)
      B[u][kv] = gok ? make_float2(B[u][kv].x * ig, B[u][kv].y * ig) : make_float2(0.f, 0.f);
  }
  if (fail) return fail;
  // smallest failing k over the group (fixed-order scan of the published gammas)
  int info = 0;
  for (int k = 0; k < S; ++k)
    if (!finite_pos(sh.gam[k])) {
      info = -(k + 1);
      break;
    }
  return info;
}

// Choose the group layout for N (grid PR x PC, register blocks MR x MC) and S (SC).
// K2 kernel: `units` matrices [units][N][N] -> weights [units][S][N], gamma, info.
template <class CF>
__global__ void __launch_bounds__(256, (CF::SC >= 4 || CF::MR * CF::MC > 56) ? 1 : 2) solve_kernel(int N, int S, long long units, const float2* __restrict__ cov,
                                                     const float2* __restrict__ steer, float2* __restrict__ wout,
                                                     float* __restrict__ gout, int32_t* __restrict__ info) {
  constexpr int G = CF::G, PR = CF::PR, PC = CF::PC, MR = CF::MR, MC = CF::MC, SC = CF::SC;
  extern __shared__ __align__(128) unsigned char smem[];
  const int ngroups = blockDim.x / G;
  const int grp = threadIdx.x / G, gl = threadIdx.x - grp * G;
  SolveShared<CF>* shs = reinterpret_cast<SolveShared<CF>*>(smem);
  SolveShared<CF>& sh = shs[grp];
  float2* wst = reinterpret_cast<float2*>(smem + ngroups * sizeof(SolveShared<CF>)) + (size_t)grp * S * N;
  const int p = gl / PC, q = gl - (gl / PC) * PC;
  const int bar_id = 1 + grp;
  // groups in one warp must run the same trip count: iterate over warp-uniform bases
  constexpr int GPW = G < 32 ? 32 / G : 1;  // groups per warp
  const int wgrp0 = (grp / GPW) * GPW;       // first group of this warp
  const long long stride = (long long)gridDim.x * ngroups;
  for (long long base = (long long)blockIdx.x * ngroups + wgrp0; base < units; base += stride) {
    const long long uidx = base + (grp - wgrp0);
    const bool valid = uidx < units;
    const long long uu = valid ? uidx : units - 1;  // clamp: compute a duplicate, store nothing
    const float2* Rg = cov + uu * N * N;
    float2 A[MR][MC], B[MR][SC];
#pragma unroll
    for (int v = 0; v < MC; ++v)
#pragma unroll
      for (int u = CF::umin(v); u < MR; ++u) {
        const int i = PR * u + p, l = PC * v + q;
        A[u][v] = (i < N && l <= i) ? Rg[i * N + l] : make_float2(0.f, 0.f);
      }
#pragma unroll
    for (int u = 0; u < MR; ++u)
#pragma unroll
      for (int kv = 0; kv < SC; ++kv) {
        const int i = PR * u + p, k = PC * kv + q;
        B[u][kv] = (i < N && k < S) ? steer[k * N + i] : make_float2(0.f, 0.f);
      }
    const int inf = group_chol_solve<CF>(N, S, A, B, sh, gl, bar_id);
    // stage w [S][N] in shared memory, then coalesced store
#pragma unroll
    for (int u = 0; u < MR; ++u)
#pragma unroll
      for (int kv = 0; kv < SC; ++kv) {
        const int i = PR * u + p, k = PC * kv + q;
        if (i < N && k < S) wst[k * N + i] = B[u][kv];
      }
    group_sync<G>(bar_id);
    if (valid) {
      float2* Wg = wout + uu * S * N;
      for (int idx = gl; idx < S * N; idx += G) Wg[idx] = wst[idx];
      if (gout)
        for (int k = gl; k < S; k += G) gout[uu * S + k] = (inf > 0) ? 0.f : (finite_pos(sh.gam[k]) ? sh.gam[k] : 0.f);
      if (gl == 0) info[uu] = inf;
    }
    group_sync<G>(bar_id);
  }
}


// ---- host-side selection ---------------------------------------------------
struct SolveSel {
  int id;       // instantiation id
  int G;        // lanes per matrix
  size_t shared_bytes;  // per group: SolveShared
};

using SolveCfg0 = SolveCfg<2, 4, 4, 2, 1>;
using SolveCfg1 = SolveCfg<2, 4, 4, 2, 2>;
using SolveCfg2 = SolveCfg<2, 4, 4, 2, 4>;
using SolveCfg3 = SolveCfg<2, 4, 4, 2, 8>;
using SolveCfg4 = SolveCfg<4, 4, 3, 3, 1>;
using SolveCfg5 = SolveCfg<4, 4, 3, 3, 2>;
using SolveCfg6 = SolveCfg<4, 4, 3, 3, 4>;
using SolveCfg7 = SolveCfg<4, 4, 3, 3, 8>;
using SolveCfg8 = SolveCfg<4, 4, 4, 4, 1>;
using SolveCfg9 = SolveCfg<4, 4, 4, 4, 2>;
using SolveCfg10 = SolveCfg<4, 4, 4, 4, 4>;
using SolveCfg11 = SolveCfg<4, 4, 4, 4, 8>;
using SolveCfg12 = SolveCfg<4, 8, 6, 3, 1>;
using SolveCfg13 = SolveCfg<4, 8, 6, 3, 2>;
using SolveCfg14 = SolveCfg<4, 8, 6, 3, 4>;
using SolveCfg15 = SolveCfg<4, 8, 8, 4, 1>;
using SolveCfg16 = SolveCfg<4, 8, 8, 4, 2>;
using SolveCfg17 = SolveCfg<4, 8, 8, 4, 4>;
using SolveCfg18 = SolveCfg<8, 8, 6, 6, 1>;
using SolveCfg19 = SolveCfg<8, 8, 6, 6, 2>;
using SolveCfg20 = SolveCfg<8, 8, 6, 6, 4>;
using SolveCfg21 = SolveCfg<8, 8, 7, 7, 1>;
using SolveCfg22 = SolveCfg<8, 8, 7, 7, 2>;
using SolveCfg23 = SolveCfg<8, 8, 7, 7, 4>;
using SolveCfg24 = SolveCfg<8, 8, 8, 8, 1>;
using SolveCfg25 = SolveCfg<8, 8, 8, 8, 2>;
using SolveCfg26 = SolveCfg<8, 8, 8, 8, 4>;

#define STAPK_SOLVE_CFGS(X) \
  X(0, SolveCfg0) \
  X(1, SolveCfg1) \
  X(2, SolveCfg2) \
  X(3, SolveCfg3) \
  X(4, SolveCfg4) \
  X(5, SolveCfg5) \
  X(6, SolveCfg6) \
  X(7, SolveCfg7) \
  X(8, SolveCfg8) \
  X(9, SolveCfg9) \
  X(10, SolveCfg10) \
  X(11, SolveCfg11) \
  X(12, SolveCfg12) \
  X(13, SolveCfg13) \
  X(14, SolveCfg14) \
  X(15, SolveCfg15) \
  X(16, SolveCfg16) \
  X(17, SolveCfg17) \
  X(18, SolveCfg18) \
  X(19, SolveCfg19) \
  X(20, SolveCfg20) \
  X(21, SolveCfg21) \
  X(22, SolveCfg22) \
  X(23, SolveCfg23) \
  X(24, SolveCfg24) \
  X(25, SolveCfg25) \
  X(26, SolveCfg26)

inline int sc_index(int S, int PC) {
  const int sc = (S + PC - 1) / PC;
  return sc <= 1 ? 0 : sc <= 2 ? 1 : sc <= 4 ? 2 : 3;
}

// false if (N, S) has no instantiation (N > 64 or S > capacity)
inline bool solve_select(int N, int S, SolveSel* s) {
  int id = -1;
  if (N <= 8) id = 0 + sc_index(S, 4);
  else if (N <= 12) id = 4 + sc_index(S, 4);
  else if (N <= 16) id = 8 + sc_index(S, 4);
  else if (N <= 24) id = (S <= 32) ? 12 + sc_index(S, 8) : -1;
  else if (N <= 32) id = (S <= 32) ? 15 + sc_index(S, 8) : -1;
  else if (N <= 48) id = 18 + sc_index(S, 8);
  else if (N <= 56) id = 21 + sc_index(S, 8);
  else if (N <= 64) id = 24 + sc_index(S, 8);
  if (id < 0) return false;
  if ((id >= 12) && sc_index(S, 8) > 2) return false;
  if (const char* e = getenv("STAP_SOLVE_ID")) {  // developer A/B knob: force a compatible layout
    const int f = atoi(e);
    if (f >= 0 && f <= 26) id = f;
  }
  switch (id) {
#define X(I, CFT) \
  case I: s->id = I; s->G = CFT::G; s->shared_bytes = sizeof(SolveShared<CFT>); break;
    STAPK_SOLVE_CFGS(X)
#undef X
    default: return false;
  }
  return true;
}

inline size_t solve_smem_bytes(const SolveSel& s, int groups, int N, int S) {
  return (size_t)groups * s.shared_bytes + (size_t)groups * S * N * 8;
}

inline void solve_set_attr(const SolveSel& s, size_t smem) {
  switch (s.id) {
#define X(I, CFT) \
  case I: cudaFuncSetAttribute(solve_kernel<CFT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); break;
    STAPK_SOLVE_CFGS(X)
#undef X
  }
}

inline void solve_launch(const SolveSel& s, int grid, int threads, size_t smem, cudaStream_t st, int N, int S,
                         long long units, const float2* cov, const float2* steer, float2* w, float* g, int32_t* info) {
  switch (s.id) {
#define X(I, CFT) \
  case I: solve_kernel<CFT><<<grid, threads, smem, st>>>(N, S, units, cov, steer, w, g, info); break;
    STAPK_SOLVE_CFGS(X)
#undef X
  }
}

}  // namespace stapk

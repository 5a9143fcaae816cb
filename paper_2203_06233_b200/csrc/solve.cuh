// solve.cuh -- K2: batched Hermitian Cholesky + forward/back solves -> MVDR weights.
//
// Method (include/stap.h; readings c-9, c-10, c-11): R = L L^H with L lower and a
// real positive diagonal; y_k = L^-1 s_k; gamma_k = ||y_k||^2; v_k = L^-H y_k
// (= R^-1 s_k); w_k = v_k / gamma_k.  A non-positive / non-finite pivot j sets
// info = j+1 and zeroes the unit's weights; a bad gamma_k sets info = -(k+1)
// for the smallest such k and zeroes w_k.
//
// Design (v1): one warp per matrix, the matrix resident in shared memory.
//  - Cholesky, left-looking by columns: lane owns rows i = lane, lane + 32; for
//    column j every owned row i >= j forms x_i = R[i][j] - sum_{m<j} L[i][m] conj(L[j][m])
//    (L[j][m] is a broadcast read), the pivot x_j is shuffled from its owner,
//    then L[i][j] = x_i / sqrt(x_j).  Row stride N+1 complex keeps the per-lane
//    row reads on distinct banks.
//  - Solves: lane k owns right-hand side k (S <= 32); y / v live in shared
//    memory [i][k] (row stride YS >= S, consecutive lanes on consecutive words),
//    L is read by broadcast.
#pragma once
#include "common.cuh"

namespace stapk {

__host__ __device__ inline int solve_ld(int N) { return N + 1; }

// Warp-cooperative factor + solve.  On entry L[i*LD + l] (l <= i) holds the lower
// triangle of R.  steer: [S][N] (shared or global).  On return Y[i*YS + k] holds
// w_k[i] (0 for failed k / failed unit; columns S..YS-1 untouched) and, for
// lane k < S, *gamma_lane = gamma_k (0 if failed).  Returns info (same on all lanes).
__device__ __forceinline__ int warp_chol_solve(int N, int S, int YS, float2* L, float2* Y,
                                               const float2* steer, float* gamma_lane) {
  const int lane = threadIdx.x & 31;
  const int LD = solve_ld(N);
  int fail = 0;
  for (int j = 0; j < N; ++j) {
    float2 x0 = make_float2(0.f, 0.f), x1 = make_float2(0.f, 0.f);
    const int i0 = lane, i1 = lane + 32;
    if (i0 >= j && i0 < N) {
      x0 = L[i0 * LD + j];
      for (int m = 0; m < j; ++m) cmsub_conjb(x0, L[i0 * LD + m], L[j * LD + m]);
    }
    if (i1 >= j && i1 < N) {
      x1 = L[i1 * LD + j];
      for (int m = 0; m < j; ++m) cmsub_conjb(x1, L[i1 * LD + m], L[j * LD + m]);
    }
    const float xj = __shfl_sync(0xffffffffu, j < 32 ? x0.x : x1.x, j & 31);
    if (!finite_pos(xj)) {
      fail = j + 1;
      break;
    }
    const float ljj = sqrtf(xj);
    const float r = 1.0f / ljj;
    __syncwarp();
    if (i0 == j) L[j * LD + j] = make_float2(ljj, 0.f);
    else if (i0 > j && i0 < N) L[i0 * LD + j] = make_float2(x0.x * r, x0.y * r);
    if (i1 == j) L[j * LD + j] = make_float2(ljj, 0.f);
    else if (i1 > j && i1 < N) L[i1 * LD + j] = make_float2(x1.x * r, x1.y * r);
    __syncwarp();
  }
  const int k = lane;
  const bool kact = k < S;
  if (fail) {
    for (int idx = lane; idx < N * YS; idx += 32) Y[idx] = make_float2(0.f, 0.f);
    if (kact) *gamma_lane = 0.f;
    __syncwarp();
    return fail;
  }
  // forward: y_i = (s_i - sum_{m<i} L[i][m] y_m) / L[i][i]
  float g = 0.f;
  if (kact) {
    for (int i = 0; i < N; ++i) {
      float2 x = steer[k * N + i];
      for (int m = 0; m < i; ++m) cmsub(x, L[i * LD + m], Y[m * YS + k]);
      const float r = 1.0f / L[i * LD + i].x;
      x.x *= r;
      x.y *= r;
      Y[i * YS + k] = x;
      g = fmaf(x.x, x.x, g);
      g = fmaf(x.y, x.y, g);
    }
  }
  const bool gok = finite_pos(g);
  if (kact) {
    if (gok) {
      // backward: v_i = (y_i - sum_{m>i} conj(L[m][i]) v_m) / L[i][i], in place
      for (int i = N - 1; i >= 0; --i) {
        float2 x = Y[i * YS + k];
        for (int m = i + 1; m < N; ++m) cmsub_conja(x, L[m * LD + i], Y[m * YS + k]);
        const float r = 1.0f / L[i * LD + i].x;
        Y[i * YS + k] = make_float2(x.x * r, x.y * r);
      }
      const float ig = 1.0f / g;
      for (int i = 0; i < N; ++i) {
        const float2 v = Y[i * YS + k];
        Y[i * YS + k] = make_float2(v.x * ig, v.y * ig);
      }
    } else {
      for (int i = 0; i < N; ++i) Y[i * YS + k] = make_float2(0.f, 0.f);
    }
    *gamma_lane = gok ? g : 0.f;
  }
  const unsigned bad = __ballot_sync(0xffffffffu, kact && !gok);
  __syncwarp();
  return bad ? -(__ffs(bad)) : 0;
}

__host__ inline size_t solve_warp_smem_bytes(int N, int S) {
  return ((size_t)N * solve_ld(N) + (size_t)N * S) * 8;
}

// `units` matrices back to back ([units][N][N]); weights [units][S][N]; gamma [units][S]; info [units].
__global__ void __launch_bounds__(256) solve_kernel(int N, int S, long long units,
                                                     const float2* __restrict__ cov,
                                                     const float2* __restrict__ steer,
                                                     float2* __restrict__ wout, float* __restrict__ gout,
                                                     int32_t* __restrict__ info) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int LD = solve_ld(N);
  float2* base = reinterpret_cast<float2*>(smem) + (size_t)warp * ((size_t)N * LD + (size_t)N * S);
  float2* L = base;                   // [N][LD]
  float2* Y = base + (size_t)N * LD;  // [N][S]

  for (long long u = (long long)blockIdx.x * nwarps + warp; u < units; u += (long long)gridDim.x * nwarps) {
    const float2* Rg = cov + u * N * N;
    for (int idx = lane; idx < N * N; idx += 32) {
      const int i = idx / N, l = idx - i * N;
      if (l <= i) L[i * LD + l] = Rg[idx];
    }
    __syncwarp();
    float g = 0.f;
    const int inf = warp_chol_solve(N, S, S, L, Y, steer, &g);
    if (gout && lane < S) gout[u * S + lane] = g;
    float2* Wg = wout + u * S * N;
    for (int idx = lane; idx < S * N; idx += 32) {
      const int kk = idx / N, i = idx - kk * N;
      Wg[idx] = Y[i * S + kk];
    }
    if (lane == 0) info[u] = inf;
    __syncwarp();
  }
}

}  // namespace stapk

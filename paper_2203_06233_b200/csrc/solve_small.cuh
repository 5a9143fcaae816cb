// solve_small.cuh -- K2 for N <= 16 (the staged path uses it for N <= 12, the fused kernel
// at N = 4 and 12; chol.cuh takes 13 <= N <= 16): Cholesky + forward/back solves, fully
// register-resident, compile-time N.
//
// Method: as chol.cuh (readings c-9, c-10, c-11).
//
// Layout: a segment of LANES lanes (16 -> two matrices per warp when S <= 16,
// else 32) owns one matrix.
//   Cholesky, right-looking: lane i holds row i of R in registers; step j
//   broadcasts the pivot and then each scaled L[l][j] (l > j) with segment
//   shuffles, every lane applying the rank-1 update to its own row (entries of
//   the upper triangle are updated too -- they are never read).  The pivots'
//   reciprocals stay in registers of every lane.
//   L is published once to shared memory; lane k then owns right-hand side k:
//   y = L^-1 s_k and v = L^-H y with y fully in registers (compile-time
//   indices), L read by broadcast loads.
// Small matrices are latency- and overhead-bound, not FMA-bound: this layout
// has no per-step barrier at all and no predicated FMA.
#pragma once
#include "common.cuh"

namespace stapk {

template <int N>
struct alignas(16) SmallShared {
  static constexpr int LD = (N + 3) & ~1;  // even row stride >= N+2: rows 16-byte aligned, pairs in bounds
  float2 L[N][LD];  // L (row i holds L[i][m], m <= i)
  float2 U[N][LD];  // U = L^H (row i holds conj(L[m][i]), m >= i) for the back solve
  float rd[N];      // 1 / L[i][i]
};

template <int N, int LANES>
__device__ __forceinline__ float2 seg_shfl(float2 v, int src) {
  return make_float2(__shfl_sync(0xffffffffu, v.x, src, LANES), __shfl_sync(0xffffffffu, v.y, src, LANES));
}

// On entry lane i (< N) of the segment holds row i of R in A[0..N) (entries l <= i
// must be valid); steer = [S][N] steering set.  On return lane k holds w_k in Y
// (zero if the unit or k failed) and *gamma = gamma_k; returns info (same on all
// lanes of the segment).  sl = lane index within the segment.  Y is loaded only
// after the factorisation so that A and Y are never live together.
template <int N, int LANES>
__device__ __forceinline__ int small_chol_solve(int S, float2 (&A)[N], const float2* __restrict__ steer,
                                                float2 (&Y)[N], SmallShared<N>& sh, int sl, float* gamma) {
  int fail = 0;
  // Branch-free steps (selects, not if/else): the segment shuffles then sit in
  // provably convergent code and compile to bare SHFLs (no convergence loops).
#pragma unroll
  for (int j = 0; j < N; ++j) {
    float x = __shfl_sync(0xffffffffu, A[j].x, j, LANES);
    const bool ok = finite_pos(x);
    fail = (!ok && !fail) ? j + 1 : fail;
    x = ok ? x : 1.0f;
    const float r = rsqrtf(x);  // one MUFU on the pivot chain
    const float d = x * r;
    if (sl == j) sh.rd[j] = r;
    const float2 a = A[j];
    A[j] = sl > j ? make_float2(a.x * r, a.y * r) : (sl == j ? make_float2(d, 0.f) : a);
#pragma unroll
    for (int l = j + 1; l < N; ++l) {
      const float2 Llj = seg_shfl<N, LANES>(A[j], l);
      cmsub_conjb(A[l], A[j], Llj);  // row sl: A[sl][l] -= L[sl][j] conj(L[l][j]); rows < l are never read
    }
  }
  // publish L (lower triangle)
  if (sl < N) {
#pragma unroll
    for (int l = 0; l < N; ++l)
      if (l <= sl) {
        sh.L[sl][l] = A[l];
        sh.U[l][sl] = make_float2(A[l].x, -A[l].y);
      }
  }
  __syncwarp();
  {
    const int k = sl < S ? sl : 0;
#pragma unroll
    for (int i = 0; i < N; ++i) Y[i] = __ldg(steer + k * N + i);
  }
  // forward: y_i = (s_i - sum_{m<i} L[i][m] y_m) / L[i][i]; row i of L read as pairs
#pragma unroll
  for (int i = 0; i < N; ++i) {
    float2 e = make_float2(0.f, 0.f);  // odd-m partial sum: halves the dependent chain
#pragma unroll
    for (int m = 0; m + 1 < i; m += 2) {
      const float4 l2 = *reinterpret_cast<const float4*>(&sh.L[i][m]);
      cmsub2(Y[i], make_float2(l2.x, l2.y), Y[m]);
      cmsub2(e, make_float2(l2.z, l2.w), Y[m + 1]);
    }
    if (i & 1) cmsub2(Y[i], sh.L[i][i - 1], Y[i - 1]);
    Y[i].x = (Y[i].x + e.x) * sh.rd[i];
    Y[i].y = (Y[i].y + e.y) * sh.rd[i];
    asm volatile("" ::: "memory");  // keep each row's loads next to their use (register pressure)
  }
  float g = 0.f;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    g = fmaf(Y[i].x, Y[i].x, g);
    g = fmaf(Y[i].y, Y[i].y, g);
  }
  // backward: v_i = (y_i - sum_{m>i} conj(L[m][i]) v_m) / L[i][i]
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    // v_i -= sum_{m>i} U[i][m] v_m, row i of U read as pairs
    float2 e = make_float2(0.f, 0.f);
    if ((i + 1) & 1) {
      if (i + 1 < N) cmsub2(Y[i], sh.U[i][i + 1], Y[i + 1]);
    }
#pragma unroll
    for (int m = ((i + 2) & ~1); m + 1 < N; m += 2) {
      const float4 u2 = *reinterpret_cast<const float4*>(&sh.U[i][m]);
      cmsub2(Y[i], make_float2(u2.x, u2.y), Y[m]);
      cmsub2(e, make_float2(u2.z, u2.w), Y[m + 1]);
    }
    if ((N - ((i + 2) & ~1)) & 1) {
      if (N - 1 > i) cmsub2(Y[i], sh.U[i][N - 1], Y[N - 1]);
    }
    Y[i].x = (Y[i].x + e.x) * sh.rd[i];
    Y[i].y = (Y[i].y + e.y) * sh.rd[i];
    asm volatile("" ::: "memory");
  }
  const bool kact = sl < S;
  const bool gok = finite_pos(g) && !fail;
  const float ig = gok ? 1.0f / g : 0.f;
#pragma unroll
  for (int i = 0; i < N; ++i) Y[i] = gok ? make_float2(Y[i].x * ig, Y[i].y * ig) : make_float2(0.f, 0.f);
  *gamma = gok ? g : 0.f;
  // smallest failing k of this segment
  const unsigned bad = __ballot_sync(0xffffffffu, kact && !finite_pos(g));
  const int seg0 = (threadIdx.x & 31) & ~(LANES - 1);
  const unsigned segbad = (bad >> seg0) & (LANES == 32 ? 0xffffffffu : ((1u << LANES) - 1u));
  __syncwarp();
  if (fail) return fail;
  return segbad ? -(__ffs(segbad)) : 0;
}

// K2 kernel (N <= 16): `units` matrices [units][N][N] -> weights [units][S][N].
template <int N, int LANES>
__global__ void __launch_bounds__(256, 2) solve_small_kernel(int S, long long units, const float2* __restrict__ cov,
                                                           const float2* __restrict__ steer, float2* __restrict__ wout,
                                                           float* __restrict__ gout, int32_t* __restrict__ info) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int SPW = 32 / LANES;  // segments (matrices) per warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int seg = lane / LANES, sl = lane - seg * LANES;
  SmallShared<N>& sh = reinterpret_cast<SmallShared<N>*>(smem)[warp * SPW + seg];
  const long long stride = (long long)gridDim.x * nwarps * SPW;
  for (long long base = ((long long)blockIdx.x * nwarps + warp) * SPW; base < units; base += stride) {
    const long long uidx = base + seg;
    const bool valid = uidx < units;
    const long long u = valid ? uidx : units - 1;
    float2 A[N], Y[N];
    const float2* Rg = cov + u * N * N + (long long)(sl < N ? sl : 0) * N;
#pragma unroll
    for (int l = 0; l < N; ++l) A[l] = Rg[l];
    float g;
    const int inf = small_chol_solve<N, LANES>(S, A, steer, Y, sh, sl, &g);
    if (valid) {
      if (sl < S) {
        float2* Wg = wout + (u * S + sl) * N;
#pragma unroll
        for (int i = 0; i < N; ++i) Wg[i] = Y[i];
        if (gout) gout[u * S + sl] = (inf > 0) ? 0.f : g;
      }
      if (sl == 0) info[u] = inf;
    }
  }
}

#define STAPK_SMALL_NS(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)

inline size_t solve_small_smem(int N, int lanes, int threads) {
  size_t per = 0;
#define X(NN) \
  if (N == NN) per = sizeof(SmallShared<NN>);
  STAPK_SMALL_NS(X)
#undef X
  return per * (threads / 32) * (32 / lanes);
}

inline void solve_small_set_attr(int N, int lanes, size_t smem) {
#define X(NN)                                                                                                  \
  if (N == NN) {                                                                                               \
    if (lanes == 16)                                                                                           \
      cudaFuncSetAttribute(solve_small_kernel<NN, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    else                                                                                                       \
      cudaFuncSetAttribute(solve_small_kernel<NN, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
  }
  STAPK_SMALL_NS(X)
#undef X
}

inline void solve_small_launch(int N, int lanes, int grid, int threads, size_t smem, cudaStream_t st, int S,
                               long long units, const float2* cov, const float2* steer, float2* w, float* g,
                               int32_t* info) {
#define X(NN)                                                                                         \
  if (N == NN) {                                                                                      \
    if (lanes == 16)                                                                                  \
      solve_small_kernel<NN, 16><<<grid, threads, smem, st>>>(S, units, cov, steer, w, g, info);      \
    else                                                                                              \
      solve_small_kernel<NN, 32><<<grid, threads, smem, st>>>(S, units, cov, steer, w, g, info);      \
  }
  STAPK_SMALL_NS(X)
#undef X
}

}  // namespace stapk

// chol.cuh -- K2 for N >= 13: batched Hermitian Cholesky + forward/back solves -> MVDR
// weights, one lane group (half warp, warp or warp pair) per matrix, register-resident.
//
// Method (include/stap.h; readings c-9, c-10, c-11): R = L L^H, L lower with a real
// positive diagonal; y_k = L^-1 s_k; gamma_k = ||y_k||^2; v_k = L^-H y_k (= R^-1 s_k);
// w_k = v_k / gamma_k.  A non-positive / non-finite pivot j sets info = j+1 and zeroes
// the unit's weights; a bad gamma_k sets info = -(k+1) for the smallest such k and
// zeroes w_k.
//
// Arithmetic without square roots (same mathematics, reordered scalings).  The factor is
// kept RAW: column j of the Schur complement at step j, a_j = L[:, j] * sqrt(p_j) with
// p_j the pivot.  The right-hand sides are kept raw as well, yraw_j = y_j * sqrt(p_j):
//   step j:  A[i][l] -= a_i conj(a_l) / p_j        (i >= l > j)
//            B[i][k] -= a_i yraw_j[k] / p_j        (i > j)
//   gamma_k = sum_m |yraw_m[k]|^2 / p_m
//   back:    v_i = (yraw_i - sum_{m > i} conj(a_m^{(i)}) v_m) / p_i
// where a_m^{(i)} = A[m][i] after step i (the raw column i).  Only 1/p_j is needed (one
// MUFU.RCP per step); no column or row is ever rescaled.
//
// B200 layout.  The round-1 group solver spent more issue slots on scaling, predicates,
// branches and scalar shared loads than on its FMAs (ncu: ALU 33%, LSU 35%, FMA pipe 43%).
//  - a group of G = PR x PC lanes owns one matrix; lane (p, q) holds A[i][l] for
//    i = PR*u + p, l = PC*v + q in A[u][v] (register blocks of the lower block triangle)
//    and B[i][k] for k = PC*kv + q in B[u][kv];
//  - step j: the owners of column j publish it raw into a parity buffer in shared memory
//    laid out [m % PR][m / PR] (16-byte pairs, rows padded so that the rows a warp reads
//    start on distinct banks) and the owners of row j publish yraw_j; ONE group barrier per
//    step; every lane reads its a_i and a_l by 16-byte loads, scales the a_l / yraw_j side by
//    1/p_j (FMUL2) and applies the rank-1 update with packed FFMA2 (common.cuh);
//  - no branches in a step: the partial diagonal block and the finished right-hand-side
//    rows are masked by zeroing the broadcast operand (x - a*0 == x exactly);
//  - pivots are only recorded (the info scan is one ballot after the loop): a failed unit
//    computes garbage that is then replaced by zeros, exactly the documented result.
#pragma once
#include <type_traits>

// strip the parentheses that protect a template-id with commas inside a macro argument
#define STAPK_UNPAREN_I(...) __VA_ARGS__
#define STAPK_UNPAREN STAPK_UNPAREN_I

#include "common.cuh"

namespace stapk {

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

template <int PR_, int PC_, int MR_, int MC_, int SC_, bool FULL_ = false, int BR_ = 4>
struct CholCfg {
  static constexpr int PR = PR_, PC = PC_, MR = MR_, MC = MC_, SC = SC_;
  static constexpr bool FULL = FULL_;  // unroll every step (else two steps per loop trip)
  static constexpr int BR = BR_;       // back solve: rows per group barrier (divides PR)
  static constexpr int G = PR * PC;  // lanes per matrix
  static_assert(G == 16 || G == 32 || G == 64, "a group is a half warp, a warp or a warp pair");
  static_assert(PR % PC == 0 || PC % PR == 0, "one lane-grid side divides the other");
  static_assert(SC == 1 || SC % 2 == 0, "right-hand sides move in pairs");
  static_assert(PR % 2 == 0 && PC % 2 == 0, "steps and rows are paired by buffer parity");
  static_assert(PR * MR == PC * MC, "square register tiling of the padded matrix");
  static_assert(BR >= 1 && PR % BR == 0, "back-solve row blocks tile a register row block");
  static constexpr int GPW = G < 32 ? 32 / G : 1;  // matrices per warp
  static constexpr int WPG = G > 32 ? G / 32 : 1;  // warps per matrix
  static constexpr int NMAX = (PR * MR < PC * MC) ? PR * MR : PC * MC;
  static constexpr int SMAX = PC * SC;
  static constexpr int MR2 = (MR + 1) & ~1;  // row blocks rounded up to pairs
  // first register row block that reaches column block v: PR*u + PR - 1 >= PC*v
  __host__ __device__ static constexpr int umin(int v) {
    return (PC * v - PR + 1) <= 0 ? 0 : (PC * v - PR + 1 + PR - 1) / PR;
  }
  __host__ __device__ static constexpr int umin2(int v) { return umin(v) & ~1; }  // even: 16-byte pairs
  // row stride of the column buffer (float2): >= MR2 and == 2 mod 16, so that the rows a
  // warp reads with 16-byte loads start 4 banks apart
  static constexpr int CS = MR2 <= 2 ? 2 : ((MR2 - 2 + 15) / 16) * 16 + 2;
  static_assert(PC % PR != 0 || PC / PR * (MC - 1) + (PC - 1) / PR < CS, "column entries fit a buffer row");
  // right-hand-side buffer stride per q (float2): 16-byte pairs, distinct banks across q
  static constexpr int SCP = SC == 1 ? 1 : SC == 2 ? 2 : SC + 2;
};

template <class CF>
struct alignas(16) CholShared {
  float2 col[2][CF::PR][CF::CS];  // raw column j (forward) / raw row i (back) at [m % PR][m / PR]
  float2 yb[2][CF::PC][CF::SCP];  // yraw_j (forward) at [q][kv] for k = PC*kv + q
  float2 rows[2][CF::BR][CF::PR][CF::CS];  // back solve: BR raw rows of the factor at [m % PR][m / PR]
  float2 tb[2][CF::BR][CF::PC][CF::SCP];   // back solve: their right-hand sides
  float piv[CF::NMAX];            // pivots p_j
  float gpart[CF::WPG][CF::SMAX]; // warp-pair groups: gamma partials per warp
  unsigned mask[CF::WPG];         // warp-pair groups: ballots per warp
};

// bytes per group, padded so that the two groups of a warp (G = 16) use opposite bank halves
template <class CF>
__host__ __device__ constexpr size_t chol_shared_bytes() {
  return ((sizeof(CholShared<CF>) + 127) / 128) * 128 + (CF::GPW > 1 ? 64 : 0);
}

template <int G>
__device__ __forceinline__ void chol_sync(int bar_id) {
  if constexpr (G <= 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(G) : "memory");
  }
}

__device__ __forceinline__ void st2x(float2* a, float2 x, float2 y) {
  *reinterpret_cast<float4*>(a) = make_float4(x.x, x.y, y.x, y.y);
}
__device__ __forceinline__ void ld2x(const float2* a, float2& x, float2& y) {
  const float4 v = *reinterpret_cast<const float4*>(a);
  x = make_float2(v.x, v.y);
  y = make_float2(v.z, v.w);
}
__device__ __forceinline__ float2 scale2(float2 a, float s) { return __fmul2_rn(a, make_float2(s, s)); }

// predicated shared stores / plain shared loads on 32-bit shared addresses (no branches)
__device__ __forceinline__ void sts128_if(bool c, uint32_t a, float2 x, float2 y) {
  asm volatile("{.reg .pred p; setp.ne.b32 p, %0, 0; @p st.shared.v4.f32 [%1], {%2, %3, %4, %5};}" ::"r"((int)c),
               "r"(a), "f"(x.x), "f"(x.y), "f"(y.x), "f"(y.y)
               : "memory");
}
__device__ __forceinline__ void sts64_if(bool c, uint32_t a, float2 x) {
  asm volatile("{.reg .pred p; setp.ne.b32 p, %0, 0; @p st.shared.v2.f32 [%1], {%2, %3};}" ::"r"((int)c), "r"(a),
               "f"(x.x), "f"(x.y)
               : "memory");
}
__device__ __forceinline__ void sts32_if(bool c, uint32_t a, float x) {
  asm volatile("{.reg .pred p; setp.ne.b32 p, %0, 0; @p st.shared.f32 [%1], %2;}" ::"r"((int)c), "r"(a), "f"(x)
               : "memory");
}
__device__ __forceinline__ void lds128(uint32_t a, float2& x, float2& y) {
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(x.x), "=f"(x.y), "=f"(y.x), "=f"(y.y) : "r"(a));
}
__device__ __forceinline__ float2 lds64(uint32_t a) {
  float2 x;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x.x), "=f"(x.y) : "r"(a));
  return x;
}
__device__ __forceinline__ float lds32(uint32_t a) {
  float x;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(a));
  return x;
}

// Shared-memory addressing of one group's buffers: per-lane bases, compile-time offsets.
template <class CF>
struct CholAddr {
  static constexpr uint32_t BUF = CF::PR * CF::CS * 8;   // one parity buffer of col
  static constexpr uint32_t YBUF = CF::PC * CF::SCP * 8; // one parity buffer of yb
  uint32_t col0, li, ll, yq, piv;
  __device__ __forceinline__ CholAddr(CholShared<CF>& sh, int p, int q) {
    constexpr int PR = CF::PR, PC = CF::PC, CS = CF::CS;
    col0 = smem_u32(&sh.col[0][0][0]);
    li = col0 + (uint32_t)(p * CS) * 8;  // rows PR*u + p at [p][u]
    if constexpr (PC % PR == 0)
      ll = col0 + (uint32_t)((q % PR) * CS + q / PR) * 8;
    else
      ll = col0 + (uint32_t)(q * CS) * 8;
    yq = smem_u32(&sh.yb[0][q][0]);
    piv = smem_u32(&sh.piv[0]);
  }
  // entry m = PC*v + q (the lane's column in block v), offset from ll
  __host__ __device__ static constexpr uint32_t ll_off(int v) {
    return CF::PC % CF::PR == 0 ? (uint32_t)((CF::PC / CF::PR) * v) * 8
                                : (uint32_t)(((CF::PC * v) % CF::PR) * CF::CS + (CF::PC * v) / CF::PR) * 8;
  }
  // entry m (runtime) of buffer b
  __device__ __forceinline__ uint32_t at(int b, int m) const {
    return col0 + (uint32_t)b * BUF + (uint32_t)((m % CF::PR) * CF::CS + m / CF::PR) * 8;
  }
};

// Up to four predicated 16-byte shared stores at a, a+16, ... under ONE predicate (one setp).
template <int NP>
__device__ __forceinline__ void sts128n_if(bool c, uint32_t a, const float2* x) {
  static_assert(NP >= 1 && NP <= 4, "1..4 pairs");
  if constexpr (NP == 1) {
    sts128_if(c, a, x[0], x[1]);
  } else if constexpr (NP == 2) {
    asm volatile(
        "{.reg .pred p; setp.ne.b32 p, %0, 0;\n"
        "@p st.shared.v4.f32 [%1], {%2, %3, %4, %5};\n"
        "@p st.shared.v4.f32 [%1+16], {%6, %7, %8, %9};}" ::"r"((int)c),
        "r"(a), "f"(x[0].x), "f"(x[0].y), "f"(x[1].x), "f"(x[1].y), "f"(x[2].x), "f"(x[2].y), "f"(x[3].x), "f"(x[3].y)
        : "memory");
  } else if constexpr (NP == 3) {
    asm volatile(
        "{.reg .pred p; setp.ne.b32 p, %0, 0;\n"
        "@p st.shared.v4.f32 [%1], {%2, %3, %4, %5};\n"
        "@p st.shared.v4.f32 [%1+16], {%6, %7, %8, %9};\n"
        "@p st.shared.v4.f32 [%1+32], {%10, %11, %12, %13};}" ::"r"((int)c),
        "r"(a), "f"(x[0].x), "f"(x[0].y), "f"(x[1].x), "f"(x[1].y), "f"(x[2].x), "f"(x[2].y), "f"(x[3].x), "f"(x[3].y),
        "f"(x[4].x), "f"(x[4].y), "f"(x[5].x), "f"(x[5].y)
        : "memory");
  } else {
    asm volatile(
        "{.reg .pred p; setp.ne.b32 p, %0, 0;\n"
        "@p st.shared.v4.f32 [%1], {%2, %3, %4, %5};\n"
        "@p st.shared.v4.f32 [%1+16], {%6, %7, %8, %9};\n"
        "@p st.shared.v4.f32 [%1+32], {%10, %11, %12, %13};\n"
        "@p st.shared.v4.f32 [%1+48], {%14, %15, %16, %17};}" ::"r"((int)c),
        "r"(a), "f"(x[0].x), "f"(x[0].y), "f"(x[1].x), "f"(x[1].y), "f"(x[2].x), "f"(x[2].y), "f"(x[3].x), "f"(x[3].y),
        "f"(x[4].x), "f"(x[4].y), "f"(x[5].x), "f"(x[5].y), "f"(x[6].x), "f"(x[6].y), "f"(x[7].x), "f"(x[7].y)
        : "memory");
  }
}

// Owners of column block v publish their raw column (rows PR*u + p, u >= umin2(v)) into
// buffer b: contiguous 16-byte pairs under one predicate.
template <class CF>
__device__ __forceinline__ void chol_publish_col(bool own, const CholAddr<CF>& ad, int b, int v,
                                                 const float2 (&A)[CF::MR][CF::MC]) {
  constexpr int MR = CF::MR;
  const int u0 = CF::umin2(v);
  const int n = MR - u0;  // entries to publish (an odd count pads with its neighbour slot)
  float2 x[CF::MR2 + 8];
#pragma unroll
  for (int u = 0; u < CF::MR2 + 8; ++u) x[u] = (u0 + u < MR) ? A[u0 + u < MR ? u0 + u : 0][v] : make_float2(0.f, 0.f);
  const uint32_t a = ad.li + (uint32_t)b * CholAddr<CF>::BUF + (uint32_t)u0 * 8;
  const int np = (n + 1) / 2;
  if (np >= 4) {
    sts128n_if<4>(own, a, x);
    if (np - 4 >= 4) sts128n_if<4>(own, a + 64, x + 8);
    else if (np - 4 == 3) sts128n_if<3>(own, a + 64, x + 8);
    else if (np - 4 == 2) sts128n_if<2>(own, a + 64, x + 8);
    else if (np - 4 == 1) sts128n_if<1>(own, a + 64, x + 8);
  } else if (np == 3) {
    sts128n_if<3>(own, a, x);
  } else if (np == 2) {
    sts128n_if<2>(own, a, x);
  } else if (np == 1) {
    sts128n_if<1>(own, a, x);
  }
}

// Owners of right-hand-side row held in B[u] publish it into yb buffer b.
template <class CF>
__device__ __forceinline__ void chol_publish_rhs(bool own, const CholAddr<CF>& ad, int b, const float2 (&Bu)[CF::SC]) {
  const uint32_t a = ad.yq + (uint32_t)b * CholAddr<CF>::YBUF;
  if constexpr (CF::SC == 1) {
    sts64_if(own, a, Bu[0]);
  } else {
#pragma unroll
    for (int kv = 0; kv < CF::SC; kv += 2) sts128_if(own, a + kv * 8, Bu[kv], Bu[kv + 1]);
  }
}

// One matrix per group.  On entry A holds R in the lane's register blocks, padded to NMAX with
// the identity (entries with i or l >= N: 1 on the diagonal, 0 elsewhere; entries above the
// diagonal may hold R's upper triangle or zero -- never read as results), B[u][kv] = s_k[i]
// (0 outside i < N, k < S).  The padding rows factor to themselves and solve to zero, so every
// step runs over the compile-time NMAX.  On return B[u][kv] = w_k[i]
// (0 for a failed k or unit) and gam[kv] = gamma_k for k = PC*kv + q; returns info (the
// same on every lane of the group).
template <class CF>
__device__ __forceinline__ int chol_solve_group(int N, int S, float2 (&A)[CF::MR][CF::MC], float2 (&B)[CF::MR][CF::SC],
                                                CholShared<CF>& sh, int gl, int bar_id, float (&gam)[CF::SC]) {
  constexpr int PR = CF::PR, PC = CF::PC, MR = CF::MR, MC = CF::MC, SC = CF::SC, G = CF::G;
  using AD = CholAddr<CF>;
  const int p = gl / PC, q = gl - (gl / PC) * PC;
  const AD ad(sh, p, q);

  // ---- publish column 0 and yraw_0
  chol_publish_col<CF>(q == 0, ad, 0, 0, A);
  chol_publish_rhs<CF>(p == 0, ad, 0, B[0]);
  chol_sync<G>(bar_id);

  // ---- Cholesky + forward solve, right-looking, one group barrier per step, over the
  // NMAX (padded) steps.  Step j = PC*v + qq reads parity buffer j & 1 (PC*v is even) and
  // publishes column j+1; CF::FULL unrolls every step (all offsets, publishing lanes and
  // masks compile-time), else two steps per loop trip with the last two steps of a column
  // block peeled (the buffer parity and the publishing block stay compile-time).
#pragma unroll
  for (int v = 0; v < MC; ++v) {
    auto step = [&](int bp, int qq, bool last) __attribute__((always_inline)) {
      const int j = PC * v + qq;
      const float pv = lds32(ad.at(bp, j));
      if (gl == 0) sh.piv[j] = pv;
      const float r2 = rcp_approx(pv);
      // a_l for the lane's columns l = PC*v2 + q, scaled by 1/p_j; block v masked to l > j
      float2 Ll[MC + 1];
      if constexpr (PR == PC) {
#pragma unroll
        for (int v2 = v & ~1; v2 < MC; v2 += 2) lds128(ad.ll + bp * AD::BUF + AD::ll_off(v2), Ll[v2], Ll[v2 + 1]);
      } else {
#pragma unroll
        for (int v2 = v; v2 < MC; ++v2) Ll[v2] = lds64(ad.ll + bp * AD::BUF + AD::ll_off(v2));
      }
      float2 yk[SC + 1];
      if constexpr (SC == 1) {
        yk[0] = lds64(ad.yq + bp * AD::YBUF);
      } else {
#pragma unroll
        for (int kv = 0; kv < SC; kv += 2) lds128(ad.yq + bp * AD::YBUF + kv * 8, yk[kv], yk[kv + 1]);
      }
      // a_i for the lane's rows i = PR*u + p (raw), 16-byte pairs
      float2 Li[CF::MR2];
#pragma unroll
      for (int u = CF::umin2(v); u < MR; u += 2) lds128(ad.li + bp * AD::BUF + u * 8, Li[u], Li[u + 1]);
      Ll[v] = scale2(Ll[v], q > qq ? r2 : 0.f);  // block v: only columns l > j change
#pragma unroll
      for (int v2 = v + 1; v2 < MC; ++v2) Ll[v2] = scale2(Ll[v2], r2);
#pragma unroll
      for (int kv = 0; kv < SC; ++kv) yk[kv] = scale2(yk[kv], r2);
      // rank-1 update of the trailing matrix: A -= a_i conj(a_l) / p_j
#pragma unroll
      for (int v2 = v; v2 < MC; ++v2) {
#pragma unroll
        for (int u = CF::umin(v2); u < MR; ++u) cmsub_conjb2(A[u][v2], Li[u], Ll[v2]);
      }
      // right-hand sides of rows i > j: B -= a_i yraw_j / p_j (rows <= j masked)
#pragma unroll
      for (int u = CF::umin(v); u < MR; ++u) {
        float2 li = Li[u];
        if (PR * u <= PC * v + PC - 1) li = (PR * u + p > j) ? li : make_float2(0.f, 0.f);
#pragma unroll
        for (int kv = 0; kv < SC; ++kv) cmsub2(B[u][kv], li, yk[kv]);
      }
      // publish column j+1 (raw) and yraw_{j+1} into the other buffer
      if (!last) {
        chol_publish_col<CF>(q == qq + 1, ad, bp ^ 1, v, A);
      } else if (v + 1 < MC) {
        chol_publish_col<CF>(q == 0, ad, bp ^ 1, v + 1, A);
      }
      if constexpr (PR == PC) {
        if (!last)
          chol_publish_rhs<CF>(p == qq + 1, ad, bp ^ 1, B[v]);
        else if (v + 1 < MR)
          chol_publish_rhs<CF>(p == 0, ad, bp ^ 1, B[v + 1]);
      } else {
        const int j1 = j + 1;
#pragma unroll
        for (int u = (PC * v) / PR; u <= (PC * v + PC) / PR && u < MR; ++u)
          chol_publish_rhs<CF>(p == j1 % PR && u == j1 / PR, ad, bp ^ 1, B[u]);
      }
      chol_sync<G>(bar_id);
    };
    if constexpr (CF::FULL) {
#pragma unroll
      for (int qq = 0; qq < PC; ++qq) step(qq & 1, qq, qq == PC - 1);
    } else {
#pragma unroll 1
      for (int q2 = 0; q2 < PC - 2; q2 += 2) {
        step(0, q2, false);
        step(1, q2 + 1, false);
      }
      step(0, PC - 2, false);
      step(1, PC - 1, true);
    }
  }

  // ---- info: the first failed pivot
  int fail = 0;
  {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j0 = 0; j0 < CF::NMAX; j0 += G) {
      const int j = j0 + gl;
      const bool bad = j < N && !finite_pos(sh.piv[j < N ? j : 0]);
      const unsigned m = __ballot_sync(0xffffffffu, bad);
      unsigned long long gm;
      if constexpr (G == 16) {
        gm = (m >> (lane & 16)) & 0xffffu;
      } else if constexpr (G == 32) {
        gm = m;
      } else {
        if (lane == 0) sh.mask[gl >> 5] = m;
        chol_sync<G>(bar_id);
        gm = (unsigned long long)sh.mask[0] | ((unsigned long long)sh.mask[1] << 32);
        chol_sync<G>(bar_id);
      }
      if (!fail && gm) fail = j0 + __ffsll((long long)gm);
    }
  }

  // ---- gamma_k = sum_m |yraw_m[k]|^2 / p_m: lane partials over its rows, fixed-order sum over p
#pragma unroll
  for (int kv = 0; kv < SC; ++kv) gam[kv] = 0.f;
#pragma unroll
  for (int u = 0; u < MR; ++u) {
    const int i = PR * u + p;
    const float ri = rcp_approx(sh.piv[i < N ? i : 0]);
#pragma unroll
    for (int kv = 0; kv < SC; ++kv) {
      const float m2 = fmaf(B[u][kv].x, B[u][kv].x, B[u][kv].y * B[u][kv].y);
      gam[kv] = i < N ? fmaf(m2, ri, gam[kv]) : gam[kv];
    }
  }
  {
    // butterfly over the lanes of a warp that share q (lane = p*PC + q)
    constexpr int PW = (G < 32 ? G : 32) / PC;  // p values per warp
#pragma unroll
    for (int kv = 0; kv < SC; ++kv)
#pragma unroll
      for (int m = PC; m < PC * PW; m <<= 1) gam[kv] += __shfl_xor_sync(0xffffffffu, gam[kv], m);
    if constexpr (CF::WPG > 1) {
      // warp-pair groups: add the two warps' sums in a fixed order
      if (p % PW == 0) {
#pragma unroll
        for (int kv = 0; kv < SC; ++kv) sh.gpart[gl >> 5][PC * kv + q] = gam[kv];
      }
      chol_sync<G>(bar_id);
#pragma unroll
      for (int kv = 0; kv < SC; ++kv) {
        float g = 0.f;
#pragma unroll
        for (int w = 0; w < CF::WPG; ++w) g += sh.gpart[w][PC * kv + q];
        gam[kv] = g;
      }
    }
  }

  // ---- back solve v = R^-1 s from the raw factor, BR rows per group barrier, from the bottom.
  // Block (ui, r0) = rows i_a = PR*ui + r0 + a, a < BR: their owners publish the raw rows and
  // current right-hand sides; every lane solves the BR x BR triangle for its k's
  //   v_a = (t_a - sum_{b > a} conj(L~[i_b][i_a]) v_b) / p_{i_a}
  // and applies the rank-BR update to its rows m < i_0:  t_m -= sum_a conj(L~[i_a][m]) v_a.
  {
    constexpr int BR = CF::BR;
    constexpr uint32_t RBUF = CF::PR * CF::CS * 8, TBUF = CF::PC * CF::SCP * 8;
    const uint32_t rows0 = smem_u32(&sh.rows[0][0][0][0]), tb0 = smem_u32(&sh.tb[0][0][q][0]);
    const uint32_t r_li = rows0 + (uint32_t)(p * CF::CS) * 8;  // rows PR*u + p of a published row
    const uint32_t r_ll = rows0 + (ad.ll - ad.col0);           // the lane's columns m = PC*v + q
#pragma unroll
    for (int ui = MR - 1; ui >= 0; --ui) {
      auto block = [&](int r0, int bb) __attribute__((always_inline)) {
        const int i0 = PR * ui + r0;
        const int a_own = p - r0;  // this lane's row of the block, if 0 <= a_own < BR
        const bool own = a_own >= 0 && a_own < BR;
        const uint32_t rsel = (uint32_t)(own ? a_own : 0) * RBUF;
        // publish the raw row and the right-hand side of the owned row
        if constexpr (PR == PC) {
#pragma unroll
          for (int v = 0; v < MC; v += 2) {
            if (ui >= CF::umin(v)) {
              const uint32_t a = r_ll + bb * BR * RBUF + rsel + AD::ll_off(v);
              if (v + 1 < MC && ui >= CF::umin(v + 1))
                sts128_if(own, a, A[ui][v], A[ui][v + 1]);
              else
                sts64_if(own, a, A[ui][v]);
            }
          }
        } else {
#pragma unroll
          for (int v = 0; v < MC; ++v)
            if (ui >= CF::umin(v)) sts64_if(own, r_ll + bb * BR * RBUF + rsel + AD::ll_off(v), A[ui][v]);
        }
        {
          const uint32_t a = tb0 + bb * BR * TBUF + (uint32_t)(own ? a_own : 0) * TBUF;
          if constexpr (SC == 1) {
            sts64_if(own, a, B[ui][0]);
          } else {
#pragma unroll
            for (int kv = 0; kv < SC; kv += 2) sts128_if(own, a + kv * 8, B[ui][kv], B[ui][kv + 1]);
          }
        }
        chol_sync<G>(bar_id);
        // the BR x BR triangle, for this lane's k's
        float2 vv[BR][SC + 1];
#pragma unroll
        for (int a = 0; a < BR; ++a) {
          const uint32_t t = tb0 + bb * BR * TBUF + a * TBUF;
          if constexpr (SC == 1) {
            vv[a][0] = lds64(t);
          } else {
#pragma unroll
            for (int kv = 0; kv < SC; kv += 2) lds128(t + kv * 8, vv[a][kv], vv[a][kv + 1]);
          }
        }
#pragma unroll
        for (int a = BR - 1; a >= 0; --a) {
          const float ra = rcp_approx(lds32(ad.piv + (i0 + a) * 4));
#pragma unroll
          for (int kv = 0; kv < SC; ++kv) vv[a][kv] = scale2(vv[a][kv], ra);
          // rows above inside the block: t_c -= conj(L~[i_a][i_c]) v_a, c < a
#pragma unroll
          for (int c = 0; c < a; ++c) {
            const int m = i0 + c;
            const float2 l = lds64(rows0 + bb * BR * RBUF + a * RBUF + (uint32_t)((m % PR) * CF::CS + m / PR) * 8);
#pragma unroll
            for (int kv = 0; kv < SC; ++kv) cmsub_conja2(vv[c][kv], l, vv[a][kv]);
          }
        }
        // owners keep their v
#pragma unroll
        for (int a = 0; a < BR; ++a)
#pragma unroll
          for (int kv = 0; kv < SC; ++kv) B[ui][kv] = (a_own == a) ? vv[a][kv] : B[ui][kv];
        // rank-BR update of the rows m < i0
        if (i0 == 0) return;
        const int ulast = r0 == 0 ? ui - 1 : ui;  // register blocks holding rows m < i0
#pragma unroll
        for (int a = 0; a < BR; ++a) {
          float2 Lm[CF::MR2];
#pragma unroll
          for (int u = 0; u <= ulast; u += 2) lds128(r_li + bb * BR * RBUF + a * RBUF + u * 8, Lm[u], Lm[u + 1]);
          if (ulast == ui) Lm[ui] = p < r0 ? Lm[ui] : make_float2(0.f, 0.f);  // rows >= i0 of block ui
#pragma unroll
          for (int u = 0; u <= ulast; ++u) {
#pragma unroll
            for (int kv = 0; kv < SC; ++kv) cmsub_conja2(B[u][kv], Lm[u], vv[a][kv]);
          }
        }
      };
      // row blocks r0 = PR - BR, ..., 0 of register row block ui; parity alternates per block
      constexpr int NB = PR / BR;
#pragma unroll
      for (int rb = NB - 1; rb >= 0; --rb) block(rb * BR, ((MR - 1 - ui) * NB + (NB - 1 - rb)) & 1);
    }
  }

  // ---- normalise: w_k = v_k / gamma_k; zero failed k or a failed unit
  int bad_k = 0;
  {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int kv = 0; kv < SC; ++kv) {
      const bool gok = finite_pos(gam[kv]) && !fail;
      const float ig = gok ? 1.0f / gam[kv] : 0.f;
#pragma unroll
      for (int u = 0; u < MR; ++u) B[u][kv] = gok ? scale2(B[u][kv], ig) : make_float2(0.f, 0.f);
      // smallest failing k = PC*kv + q (every lane of a q column holds the same gamma); the
      // lanes with p == 0 sit in the group's first warp at lane offsets q
      const int k = PC * kv + q;
      const unsigned m = __ballot_sync(0xffffffffu, p == 0 && k < S && !finite_pos(gam[kv]));
      const unsigned gm = G == 16 ? ((m >> (lane & 16)) & 0xffffu) : m;
      if (G > 32 && (gl >> 5) != 0) continue;  // the second warp of a pair has no p == 0 lanes
      if (!bad_k && gm) bad_k = PC * kv + __ffs(gm);
    }
    if constexpr (G > 32) {
      if (gl == 0) sh.mask[0] = (unsigned)bad_k;
      chol_sync<G>(bar_id);
      bad_k = (int)sh.mask[0];
    }
  }
  chol_sync<G>(bar_id);  // every lane is done with the buffers before the next matrix publishes
  if (fail) return fail;
  return bad_k ? -bad_k : 0;
}

// K2 kernel (N >= 13, see chol_select): `units` matrices [units][N][N] (full Hermitian; each lane reads the
// entries of its register blocks, so the upper entries track the Hermitian Schur complement)
// -> weights [units][S][N], gamma [units][S] (nullable), info [units].
template <class CF, int kThreads, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    chol_kernel(int N, int S, long long units, const float2* __restrict__ cov, const float2* __restrict__ steer,
                float2* __restrict__ wout, float* __restrict__ gout, int32_t* __restrict__ info) {
  constexpr int PR = CF::PR, PC = CF::PC, MR = CF::MR, MC = CF::MC, SC = CF::SC, G = CF::G;
  extern __shared__ __align__(128) unsigned char smem[];
  const int ngroups = kThreads / G;
  const int grp = threadIdx.x / G, gl = threadIdx.x - grp * G;
  const int p = gl / PC, q = gl - (gl / PC) * PC;
  CholShared<CF>& sh = *reinterpret_cast<CholShared<CF>*>(smem + (size_t)grp * chol_shared_bytes<CF>());
  const int bar_id = 1 + grp;
  const long long stride = (long long)gridDim.x * ngroups;
  for (long long base = (long long)blockIdx.x * ngroups + (grp / CF::GPW) * CF::GPW; base < units; base += stride) {
    const long long uidx = base + grp % CF::GPW;
    const bool valid = uidx < units;
    const long long uu = valid ? uidx : units - 1;  // a duplicate is computed, nothing stored
    const float2* Rg = cov + uu * N * N;
    float2 A[MR][MC], B[MR][SC];
#pragma unroll
    for (int v = 0; v < MC; ++v)
#pragma unroll
      for (int u = CF::umin(v); u < MR; ++u) {
        const int i = PR * u + p, l = PC * v + q;
        A[u][v] = (i < N && l < N) ? __ldg(Rg + i * N + l) : make_float2(i == l ? 1.f : 0.f, 0.f);
      }
#pragma unroll
    for (int u = 0; u < MR; ++u)
#pragma unroll
      for (int kv = 0; kv < SC; ++kv) {
        const int i = PR * u + p, k = PC * kv + q;
        B[u][kv] = (i < N && k < S) ? __ldg(steer + k * N + i) : make_float2(0.f, 0.f);
      }
    float gam[SC];
    const int inf = chol_solve_group<CF>(N, S, A, B, sh, gl, bar_id, gam);
    if (valid) {
      float2* Wg = wout + uu * S * N;
#pragma unroll
      for (int u = 0; u < MR; ++u)
#pragma unroll
        for (int kv = 0; kv < SC; ++kv) {
          const int i = PR * u + p, k = PC * kv + q;
          if (i < N && k < S) Wg[k * N + i] = B[u][kv];
        }
      if (gout && p == 0) {
#pragma unroll
        for (int kv = 0; kv < SC; ++kv) {
          const int k = PC * kv + q;
          if (k < S) gout[uu * S + k] = (inf > 0 || !finite_pos(gam[kv])) ? 0.f : gam[kv];
        }
      }
      if (gl == 0) info[uu] = inf;
    }
  }
}

// ---- host-side selection ---------------------------------------------------
// Instantiations (N >= 13; N <= 12 runs solve_small.cuh).  Measured on B200 (65536 large /
// 131072 medium matrices, S = 16): 4x8 lanes, 14x7 blocks, one 256-thread block per SM (8
// warps): 1.583 ms (2 x 128: 1.611 ms; 4 x 64: 1.684 ms; old 8x8 two-warp group solver 2.23 ms);
// N <= 32: 4x8 lanes, 8x4 blocks, one 512-thread block per SM (16 warps, 128 registers):
// 0.943 ms (2 x 256: 0.998 ms; 3 x 128 at 136 registers: 1.036 ms; 8 x 64: 1.055 ms; old
// 1.22).  Same warps per SM, one block: the results are bitwise those of the smaller blocks.
#define STAPK_CHOL_CFGS(X)                                      \
  X(0, (CholCfg<4, 8, 8, 4, 1, false, 2>), 128, 3)              \
  X(1, (CholCfg<4, 8, 8, 4, 2, false, 2>), 512, 1)              \
  X(2, (CholCfg<4, 8, 8, 4, 4, false, 2>), 128, 2)              \
  X(3, (CholCfg<4, 8, 14, 7, 1, false, 2>), 256, 1)             \
  X(4, (CholCfg<4, 8, 14, 7, 2, false, 2>), 256, 1)             \
  X(5, (CholCfg<8, 8, 7, 7, 4, false, 4>), 64, 4)               \
  X(6, (CholCfg<8, 8, 8, 8, 1, false, 4>), 64, 5)               \
  X(7, (CholCfg<8, 8, 8, 8, 2, false, 4>), 64, 5)               \
  X(8, (CholCfg<8, 8, 8, 8, 4, false, 4>), 64, 4)               \
  X(9, (CholCfg<4, 4, 4, 4, 1, false, 2>), 512, 1)              \
  X(10, (CholCfg<4, 4, 4, 4, 2, false, 2>), 512, 1)             \
  X(11, (CholCfg<4, 4, 4, 4, 4, false, 2>), 512, 1)             \
  X(12, (CholCfg<4, 4, 4, 4, 8, false, 2>), 512, 1)             \
  X(13, (CholCfg<4, 4, 6, 6, 2, false, 2>), 512, 1)             \
  X(14, (CholCfg<4, 4, 6, 6, 4, false, 2>), 512, 1)             \
  X(15, (CholCfg<4, 8, 10, 5, 1, false, 2>), 384, 1)            \
  X(16, (CholCfg<4, 8, 10, 5, 2, false, 2>), 384, 1)            \
  X(17, (CholCfg<4, 8, 12, 6, 1, false, 2>), 256, 1)            \
  X(18, (CholCfg<4, 8, 12, 6, 2, false, 2>), 256, 1)

struct CholSel {
  int id = -1;
  int threads = 0;     // per block
  int groups = 0;      // matrices per block
  size_t smem = 0;     // per block
  int min_blocks = 0;  // per SM (launch bounds)
};

// false if (N, S) has no instantiation here: N <= 12 (solve_small.cuh, whose arithmetic the
// fused kernel shares, so the small configuration's staged and fused paths agree to 1e-5),
// N > 64 or S > 32.  N = 13..16 (any S) and N = 17..24 with S <= 16 run half-warp groups (4x4
// lanes, two matrices per warp, the matrix padded to 16 or 24 instead of 32); measured on B200
// (262144 matrices): N = 16, S = 16 0.553 ms vs 1.052 on solve_small.cuh; N = 16, S = 32 1.23
// vs 1.83 ms; N = 24, S = 16 1.11 ms vs 1.87 on the 4x8-lane, 32-row layout; N = 20, S = 8
// 0.61 vs 1.82 ms (N = 12, S = 16 0.350 vs 0.374 ms and N = 10, S = 8 0.235 vs 0.209 ms against
// solve_small; at N = 17..24, S > 16 the 4x4 lanes spill and the 4x8 layout stays).  Likewise
// N = 33..40 and 41..48 with S <= 16 get 40- and 48-row layouts instead of 56: N = 48, S = 16
// 1.25 vs 1.66 ms; N = 40, S = 16 0.76 ms (65536 matrices).
inline bool chol_select(int N, int S, CholSel* sel) {
  int id = -1;
  const int sc = S <= 8 ? 1 : S <= 16 ? 2 : S <= 32 ? 4 : 0;
  if (N < 13 || N > 64 || !sc) return false;
  const int sc4 = S <= 4 ? 1 : S <= 8 ? 2 : S <= 16 ? 4 : 8;  // right-hand-side columns per lane (PC = 4)
  if (N <= 16) id = sc4 == 1 ? 9 : sc4 == 2 ? 10 : sc4 == 4 ? 11 : 12;
  else if (N <= 24 && sc4 <= 4) id = sc4 <= 2 ? 13 : 14;
  else if (N <= 32) id = sc == 1 ? 0 : sc == 2 ? 1 : 2;
  else if (N <= 40 && sc <= 2) id = sc == 1 ? 15 : 16;
  else if (N <= 48 && sc <= 2) id = sc == 1 ? 17 : 18;
  else if (N <= 56) id = sc == 1 ? 3 : sc == 2 ? 4 : 5;
  else id = sc == 1 ? 6 : sc == 2 ? 7 : 8;
  switch (id) {
#define X(I, CFT, TH, MB)                                      \
  case I: {                                                    \
    using CF_ = STAPK_UNPAREN CFT;                             \
    sel->id = I;                                               \
    sel->threads = TH;                                         \
    sel->groups = TH / CF_::G;                                 \
    sel->smem = (size_t)(TH / CF_::G) * chol_shared_bytes<CF_>(); \
    sel->min_blocks = MB;                                      \
    break;                                                     \
  }
    STAPK_CHOL_CFGS(X)
#undef X
    default: return false;
  }
  return true;
}

inline cudaError_t chol_set_attr(const CholSel& s) {
  switch (s.id) {
#define X(I, CFT, TH, MB) \
  case I: return cudaFuncSetAttribute(chol_kernel<STAPK_UNPAREN CFT, TH, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s.smem);
    STAPK_CHOL_CFGS(X)
#undef X
  }
  return cudaErrorInvalidValue;
}

inline void chol_launch(const CholSel& s, int grid, cudaStream_t st, int N, int S, long long units, const float2* cov,
                        const float2* steer, float2* w, float* g, int32_t* info) {
  switch (s.id) {
#define X(I, CFT, TH, MB) \
  case I: chol_kernel<STAPK_UNPAREN CFT, TH, MB><<<grid, TH, s.smem, st>>>(N, S, units, cov, steer, w, g, info); break;
    STAPK_CHOL_CFGS(X)
#undef X
  }
}

}  // namespace stapk

// chol_ws.cuh -- K2, warp-specialised variant of chol.cuh (same arithmetic, same results).
//
// chol.cuh runs one matrix per warp: the factor update, the right-hand-side update and the
// back solve issue back to back from one warp, so a matrix takes the sum of the three.
// Here a matrix is owned by a warp PAIR with split roles:
//   F (factor warp): holds A in registers (the same 4x8 lane grid and block-cyclic register
//     blocks as chol.cuh), runs the rank-1 updates A -= a_i conj(a_l)/p_j and streams each raw
//     column a_j through a ring of RD shared-memory slots; after the last column it streams the
//     raw rows of the factor (BR rows per slot) through a second ring, then loads the next
//     matrix.
//   S (solve warp): holds B (the right-hand sides) in registers, consumes the columns
//     (B -= a_i yraw_j / p_j), computes gamma and info, then consumes the rows for the back
//     solve and writes the weights.
// So the factorisation of matrix m+1 overlaps the back solve of matrix m, and the two update
// streams of one step run on two warps.  Producer/consumer progress is four monotonic
// counters per pair in shared memory (st.release / ld.acquire at CTA scope); within a warp
// the ring slots are ordered by __syncwarp.  The mathematics is chol.cuh's (see its header):
// the same raw factor, one rcp.approx per pivot, the same masks and the same summation order,
// so the weights are bitwise those of chol_kernel for the same configuration.
#pragma once
#include "chol.cuh"

namespace stapk {

template <class CF, int RD, int RDB>
struct alignas(16) WsShared {
  uint64_t cfull[RD], cempty[RD], rfull[RDB], rempty[RDB];  // ring slot mbarriers (count 1)
  float2 col[RD][CF::PR][CF::CS];             // column ring: raw column j at [m % PR][m / PR]
  float2 rows[RDB][CF::BR][CF::PR][CF::CS];   // row ring: BR raw rows of the factor
  float2 yb[2][CF::PC][CF::SCP];              // S: yraw_j at [q][kv]
  float2 tb[2][CF::BR][CF::PC][CF::SCP];      // S: back-solve right-hand sides
  float piv[CF::NMAX];                        // S: pivots of the current matrix
};

template <class CF, int RD, int RDB>
__host__ __device__ constexpr size_t ws_shared_bytes() {
  return ((sizeof(WsShared<CF, RD, RDB>) + 127) / 128) * 128;
}

__device__ __forceinline__ void st_release_s32(uint32_t a, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_s32(uint32_t a) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void ws_wait_ge(uint32_t a, int v) {
  while (ld_acquire_s32(a) < v) {
  }
}

// One warp pair per matrix, NG pairs per block: warp 2g is F, warp 2g+1 is S.
template <class CF, int NG, int kMinBlocks, int RD = 4, int RDB = 4>
__global__ void __launch_bounds__(64 * NG, kMinBlocks)
    chol_ws_kernel(int N, int S, long long units, const float2* __restrict__ cov, const float2* __restrict__ steer,
                   float2* __restrict__ wout, float* __restrict__ gout, int32_t* __restrict__ info) {
  constexpr int PR = CF::PR, PC = CF::PC, MR = CF::MR, MC = CF::MC, SC = CF::SC, BR = CF::BR, CS = CF::CS;
  constexpr int NMAX = CF::NMAX, NB = PR / BR, NBLK = MR * NB;
  static_assert(CF::G == 32 && PC % PR == 0, "one warp per role, PC a multiple of PR");
  static_assert(NMAX % RD == 0 && NBLK % RDB == 0 && (RD & (RD - 1)) == 0 && (RDB & (RDB - 1)) == 0,
                "ring slots repeat per matrix");
  static_assert(PC >= 4, "two steps per loop trip, the last two peeled");
  constexpr uint32_t BUF = PR * CS * 8, RBUF = PR * CS * 8, YBUF = PC * CF::SCP * 8, TBUF = PC * CF::SCP * 8;
  using SH = WsShared<CF, RD, RDB>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = warp >> 1;
  const bool is_f = (warp & 1) == 0;
  const int p = lane / PC, q = lane % PC;
  SH& sh = *reinterpret_cast<SH*>(smem + (size_t)grp * ws_shared_bytes<CF, RD, RDB>());
  const uint32_t col0 = smem_u32(&sh.col[0][0][0]);
  const uint32_t li = col0 + (uint32_t)(p * CS) * 8;                          // rows PR*u + p
  const uint32_t ll = col0 + (uint32_t)((q % PR) * CS + q / PR) * 8;          // columns PC*v + q
  auto ll_off = [](int v) { return (uint32_t)((PC / PR) * v) * 8; };
  auto at = [&](uint32_t base, int m) { return base + (uint32_t)((m % PR) * CS + m / PR) * 8; };
  if (lane == 0 && is_f) {
#pragma unroll
    for (int r = 0; r < RD; ++r) {
      mbar_init(&sh.cfull[r], 1);
      mbar_init(&sh.cempty[r], 1);
    }
#pragma unroll
    for (int r = 0; r < RDB; ++r) {
      mbar_init(&sh.rfull[r], 1);
      mbar_init(&sh.rempty[r], 1);
    }
  }
  // column c / row block b sit in slot c % RD / b % RDB, phase (c / RD) & 1 / (b / RDB) & 1
  auto c_free = [&](int c) { mbar_wait(&sh.cempty[c & (RD - 1)], ((c / RD) & 1) ^ 1); };
  auto c_pub = [&](int c) { mbar_arrive(&sh.cfull[c & (RD - 1)]); };
  auto c_ready = [&](int c) { mbar_wait(&sh.cfull[c & (RD - 1)], (c / RD) & 1); };
  auto c_done = [&](int c) { mbar_arrive(&sh.cempty[c & (RD - 1)]); };
  auto r_free = [&](int b) { mbar_wait(&sh.rempty[b & (RDB - 1)], ((b / RDB) & 1) ^ 1); };
  auto r_pub = [&](int b) { mbar_arrive(&sh.rfull[b & (RDB - 1)]); };
  auto r_ready = [&](int b) { mbar_wait(&sh.rfull[b & (RDB - 1)], (b / RDB) & 1); };
  auto r_done = [&](int b) { mbar_arrive(&sh.rempty[b & (RDB - 1)]); };
  asm volatile("bar.sync %0, 64;" ::"r"(1 + grp) : "memory");

  const long long stride = (long long)gridDim.x * NG;
  int cbase = 0, rbase = 0;  // global column / row-block counters of this pair
  if (is_f) {
    // =========================== F: factor warp ===========================
    for (long long uidx = (long long)blockIdx.x * NG + grp; uidx < units; uidx += stride) {
      const float2* Rg = cov + uidx * N * N;
      float2 A[MR][MC];
#pragma unroll
      for (int v = 0; v < MC; ++v)
#pragma unroll
        for (int u = CF::umin(v); u < MR; ++u) {
          const int i = PR * u + p, l = PC * v + q;
          A[u][v] = (i < N && l < N) ? __ldg(Rg + i * N + l) : make_float2(i == l ? 1.f : 0.f, 0.f);
        }
      // publish column 0 into slot 0
      c_free(cbase);
      {
        // owners q == 0 of column block 0
        const int u0 = CF::umin2(0);
        float2 x[CF::MR2 + 8];
#pragma unroll
        for (int u = 0; u < CF::MR2 + 8; ++u) x[u] = (u0 + u < MR) ? A[u0 + u < MR ? u0 + u : 0][0] : make_float2(0.f, 0.f);
        const uint32_t a = li + (uint32_t)u0 * 8;
        constexpr int np = (MR - 0 + 1) / 2;
        if constexpr (np >= 4) {
          sts128n_if<4>(q == 0, a, x);
          if constexpr (np - 4 >= 4) sts128n_if<4>(q == 0, a + 64, x + 8);
          else if constexpr (np - 4 == 3) sts128n_if<3>(q == 0, a + 64, x + 8);
          else if constexpr (np - 4 == 2) sts128n_if<2>(q == 0, a + 64, x + 8);
          else if constexpr (np - 4 == 1) sts128n_if<1>(q == 0, a + 64, x + 8);
        } else {
          sts128n_if<np>(q == 0, a, x);
        }
      }
      __syncwarp();
      if (lane == 0) c_pub(cbase);

#pragma unroll
      for (int v = 0; v < MC; ++v) {
        auto step = [&](int qq, bool last) __attribute__((always_inline)) {
          const int j = PC * v + qq;
          const uint32_t sb = (uint32_t)(j & (RD - 1)) * BUF;
          const float pv = lds32(at(col0 + sb, j));
          const float r2 = rcp_approx(pv);
          float2 Ll[MC + 1];
#pragma unroll
          for (int v2 = v; v2 < MC; ++v2) Ll[v2] = lds64(ll + sb + ll_off(v2));
          float2 Li[CF::MR2];
#pragma unroll
          for (int u = CF::umin2(v); u < MR; u += 2) lds128(li + sb + u * 8, Li[u], Li[u + 1]);
          Ll[v] = scale2(Ll[v], q > qq ? r2 : 0.f);
#pragma unroll
          for (int v2 = v + 1; v2 < MC; ++v2) Ll[v2] = scale2(Ll[v2], r2);
#pragma unroll
          for (int v2 = v; v2 < MC; ++v2) {
#pragma unroll
            for (int u = CF::umin(v2); u < MR; ++u) cmsub_conjb2(A[u][v2], Li[u], Ll[v2]);
          }
          if (last && v + 1 == MC) return;
          const int cn = cbase + j + 1;
          c_free(cn);
          // publish column j+1 into its slot
          const int vn = last ? v + 1 : v;
          const bool own = last ? (q == 0) : (q == qq + 1);
          const uint32_t sbn = (uint32_t)((j + 1) & (RD - 1)) * BUF;
          {
            const int u0 = CF::umin2(vn);
            float2 x[CF::MR2 + 8];
#pragma unroll
            for (int u = 0; u < CF::MR2 + 8; ++u)
              x[u] = (u0 + u < MR) ? A[u0 + u < MR ? u0 + u : 0][vn < MC ? vn : 0] : make_float2(0.f, 0.f);
            const uint32_t a = li + sbn + (uint32_t)u0 * 8;
            const int np = (MR - u0 + 1) / 2;
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
          __syncwarp();
          if (lane == 0) c_pub(cn);
        };
#pragma unroll 1
        for (int q2 = 0; q2 < PC - 2; q2 += 2) {
          step(q2, false);
          step(q2 + 1, false);
        }
        step(PC - 2, false);
        step(PC - 1, true);
      }
      cbase += NMAX;

      // stream the raw rows of the factor, BR per slot, from the bottom
      const uint32_t rows0 = smem_u32(&sh.rows[0][0][0][0]);
      const uint32_t r_ll = rows0 + (ll - col0);
#pragma unroll
      for (int ui = MR - 1; ui >= 0; --ui) {
#pragma unroll
        for (int rb = NB - 1; rb >= 0; --rb) {
          const int lb = (MR - 1 - ui) * NB + (NB - 1 - rb);
          const int gb = rbase + lb;
          const int a_own = p - rb * BR;
          const bool own = a_own >= 0 && a_own < BR;
          const uint32_t rsel = (uint32_t)(own ? a_own : 0) * RBUF + (uint32_t)(lb & (RDB - 1)) * BR * RBUF;
          r_free(gb);
#pragma unroll
          for (int v = 0; v < MC; ++v)
            if (ui >= CF::umin(v)) sts64_if(own, r_ll + rsel + ll_off(v), A[ui][v]);
          __syncwarp();
          if (lane == 0) r_pub(gb);
        }
      }
      rbase += NBLK;
    }
    return;
  }

  // =========================== S: solve warp ===========================
  const uint32_t yq = smem_u32(&sh.yb[0][q][0]);
  const uint32_t pivs = smem_u32(&sh.piv[0]);
  for (long long uidx = (long long)blockIdx.x * NG + grp; uidx < units; uidx += stride) {
    float2 B[MR][SC];
#pragma unroll
    for (int u = 0; u < MR; ++u)
#pragma unroll
      for (int kv = 0; kv < SC; ++kv) {
        const int i = PR * u + p, k = PC * kv + q;
        B[u][kv] = (i < N && k < S) ? __ldg(steer + k * N + i) : make_float2(0.f, 0.f);
      }
    auto pub_rhs = [&](bool own, uint32_t a, const float2(&Bu)[SC]) __attribute__((always_inline)) {
      if constexpr (SC == 1) {
        sts64_if(own, a, Bu[0]);
      } else {
#pragma unroll
        for (int kv = 0; kv < SC; kv += 2) sts128_if(own, a + kv * 8, Bu[kv], Bu[kv + 1]);
      }
    };
    pub_rhs(p == 0, yq, B[0]);
    __syncwarp();

#pragma unroll
    for (int v = 0; v < MC; ++v) {
      auto step = [&](int qq) __attribute__((always_inline)) {
        const int j = PC * v + qq;
        const int c = cbase + j;
        const int bp = qq & 1;  // PC*v is even
        c_ready(c);
        const uint32_t sb = (uint32_t)(j & (RD - 1)) * BUF;
        const float pv = lds32(at(col0 + sb, j));
        if (lane == 0) sh.piv[j] = pv;
        const float r2 = rcp_approx(pv);
        float2 yk[SC + 1];
        if constexpr (SC == 1) {
          yk[0] = lds64(yq + bp * YBUF);
        } else {
#pragma unroll
          for (int kv = 0; kv < SC; kv += 2) lds128(yq + bp * YBUF + kv * 8, yk[kv], yk[kv + 1]);
        }
        float2 Li[CF::MR2];
#pragma unroll
        for (int u = CF::umin2(v); u < MR; u += 2) lds128(li + sb + u * 8, Li[u], Li[u + 1]);
#pragma unroll
        for (int kv = 0; kv < SC; ++kv) yk[kv] = scale2(yk[kv], r2);
#pragma unroll
        for (int u = CF::umin(v); u < MR; ++u) {
          float2 lv = Li[u];
          if (PR * u <= PC * v + PC - 1) lv = (PR * u + p > j) ? lv : make_float2(0.f, 0.f);
#pragma unroll
          for (int kv = 0; kv < SC; ++kv) cmsub2(B[u][kv], lv, yk[kv]);
        }
        const int j1 = j + 1;
#pragma unroll
        for (int u = (PC * v) / PR; u <= (PC * v + PC) / PR && u < MR; ++u)
          pub_rhs(p == j1 % PR && u == j1 / PR, yq + (bp ^ 1) * YBUF, B[u]);
        __syncwarp();
        if (lane == 0) c_done(c);
      };
#pragma unroll 1
      for (int q2 = 0; q2 < PC - 2; q2 += 2) {
        step(q2);
        step(q2 + 1);
      }
      step(PC - 2);
      step(PC - 1);
    }
    cbase += NMAX;

    // ---- info: the first failed pivot (G == 32)
    int fail = 0;
#pragma unroll
    for (int j0 = 0; j0 < NMAX; j0 += 32) {
      const int j = j0 + lane;
      const bool bad = j < N && !finite_pos(sh.piv[j < N ? j : 0]);
      const unsigned m = __ballot_sync(0xffffffffu, bad);
      if (!fail && m) fail = j0 + __ffs(m);
    }
    // ---- gamma
    float gam[SC];
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
#pragma unroll
    for (int kv = 0; kv < SC; ++kv)
#pragma unroll
      for (int m = PC; m < 32; m <<= 1) gam[kv] += __shfl_xor_sync(0xffffffffu, gam[kv], m);

    // ---- back solve from the streamed rows (chol.cuh's blocked back solve)
    {
      const uint32_t rows0 = smem_u32(&sh.rows[0][0][0][0]), tb0 = smem_u32(&sh.tb[0][0][q][0]);
      const uint32_t r_li = rows0 + (uint32_t)(p * CS) * 8;
#pragma unroll
      for (int ui = MR - 1; ui >= 0; --ui) {
        auto block = [&](int rb) __attribute__((always_inline)) {
          const int r0 = rb * BR;
          const int lb = (MR - 1 - ui) * NB + (NB - 1 - rb);
          const int gb = rbase + lb;
          const int bb = lb & 1;
          const uint32_t rs = rows0 + (uint32_t)(lb & (RDB - 1)) * BR * RBUF;
          const uint32_t rsl = r_li + (uint32_t)(lb & (RDB - 1)) * BR * RBUF;
          const int i0 = PR * ui + r0;
          const int a_own = p - r0;
          const bool own = a_own >= 0 && a_own < BR;
          pub_rhs(own, tb0 + bb * BR * TBUF + (uint32_t)(own ? a_own : 0) * TBUF, B[ui]);
          r_ready(gb);
          __syncwarp();
          if (lane == 0 && lb > 0) r_done(gb - 1);  // the previous block's rows are read
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
            const float ra = rcp_approx(lds32(pivs + (i0 + a) * 4));
#pragma unroll
            for (int kv = 0; kv < SC; ++kv) vv[a][kv] = scale2(vv[a][kv], ra);
#pragma unroll
            for (int c = 0; c < a; ++c) {
              const float2 l = lds64(at(rs + a * RBUF, i0 + c));
#pragma unroll
              for (int kv = 0; kv < SC; ++kv) cmsub_conja2(vv[c][kv], l, vv[a][kv]);
            }
          }
#pragma unroll
          for (int a = 0; a < BR; ++a)
#pragma unroll
            for (int kv = 0; kv < SC; ++kv) B[ui][kv] = (a_own == a) ? vv[a][kv] : B[ui][kv];
          if (i0 == 0) return;
          const int ulast = r0 == 0 ? ui - 1 : ui;
#pragma unroll
          for (int a = 0; a < BR; ++a) {
            float2 Lm[CF::MR2];
#pragma unroll
            for (int u = 0; u <= ulast; u += 2) lds128(rsl + a * RBUF + u * 8, Lm[u], Lm[u + 1]);
            if (ulast == ui) Lm[ui] = p < r0 ? Lm[ui] : make_float2(0.f, 0.f);
#pragma unroll
            for (int u = 0; u <= ulast; ++u) {
#pragma unroll
              for (int kv = 0; kv < SC; ++kv) cmsub_conja2(B[u][kv], Lm[u], vv[a][kv]);
            }
          }
        };
#pragma unroll
        for (int rb = NB - 1; rb >= 0; --rb) block(rb);
      }
      __syncwarp();
      if (lane == 0) r_done(rbase + NBLK - 1);
    }
    rbase += NBLK;

    // ---- normalise, store
    int bad_k = 0;
#pragma unroll
    for (int kv = 0; kv < SC; ++kv) {
      const bool gok = finite_pos(gam[kv]) && !fail;
      const float ig = gok ? 1.0f / gam[kv] : 0.f;
#pragma unroll
      for (int u = 0; u < MR; ++u) B[u][kv] = gok ? scale2(B[u][kv], ig) : make_float2(0.f, 0.f);
      const int k = PC * kv + q;
      const unsigned m = __ballot_sync(0xffffffffu, p == 0 && k < S && !finite_pos(gam[kv]));
      if (!bad_k && m) bad_k = PC * kv + __ffs(m);
    }
    const int inf = fail ? fail : (bad_k ? -bad_k : 0);
    float2* Wg = wout + uidx * S * N;
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
        if (k < S) gout[uidx * S + k] = (inf > 0 || !finite_pos(gam[kv])) ? 0.f : gam[kv];
      }
    }
    if (lane == 0) info[uidx] = inf;
  }
}

}  // namespace stapk

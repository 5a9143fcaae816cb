// apply_tc.cuh -- K3 on the 5th-generation tensor cores (tcgen05.mma kind::tf32)
// with a 3xTF32 split so the result keeps FP32 accuracy.  Used by the staged path
// when S = 16, K % 64 == 0 and N <= 64 (medium / large); the SIMT apply (apply.cuh)
// covers every other shape.
//
// Method (include/stap.h; reading c-12 -- the paper shows the STAP kernel only as
// a figure, whose statement U is the 2-D x 2-D array multiply of
// PAPER.md:420-425): Y[d][k][r] = w_{d,b(r),k}^H z_{d,r}, written as one real GEMM per tile of 64 range cells of
// a unit (d, b):
//   rows    m = 2*jj + part, jj < 64 the cell, part 0 = Re z, 1 = Im z   -> M = 128
//   columns n < S: Re w_k,  n >= S: Im w_{n-S}                          -> N = 2S = 32
//   reduction i = snapshot element t*C + c, zero-padded to 8*KS         -> K = 8 per MMA
//   Out[m][n] = sum_i A[m][i] B[n][i],  A[2jj+p][i] = part_p(z_i[jj]),  B as above
//   Re Y[k][jj] = Out[2jj][k] + Out[2jj+1][S+k],  Im Y[k][jj] = Out[2jj+1][k] - Out[2jj][S+k]
// 3xTF32: x = hi + lo with hi = x as stored (the tensor core reads it truncated to TF32)
//   and lo = x - trunc_TF32(x) (exact, |lo| < 2^-10 |x|, truncated by the MMA in turn:
//   error < 2^-21 |x|);  A B ~= Ahi Bhi + Ahi Blo + Alo Bhi (dropped Alo Blo < 2^-20 |A||B|),
//   FP32 accumulation in tensor memory.
//
// Data movement (B200-first):
//   * A (the snapshots, 128 x 8KS): the N rows of a tile are T boxes of {64 cells, C
//     channels} of the cube; one thread TMA-loads them (cp.async.bulk.tensor.2d) into a
//     ring of ns shared-memory stages on mbarriers.  The two warps of TMEM lane
//     quarter q read the (cell, part) columns m = 32q + lane of the stage
//     (conflict-free), split them and write TMEM lane m (half of the k-steps each)
//     with tcgen05.st;
//     the MMA reads A from TMEM (the "TS" form), so the dominant operand needs no
//     transpose and its hi/lo copies cost no shared-memory bandwidth.
//   * B (the weights: 32 hi rows then 32 lo rows x 8KS) goes to shared memory in the
//     canonical K-major no-swizzle layout (8-row x 16-byte core matrices: LBO = 128 B between the two
//     4-element halves of an MMA k-step, SBO = 256 B between 8-row groups).
//   * Warp-specialised pipeline, two persistent CTAs per SM (10 warps and 256 TMEM
//     columns each): a producer warp issues the TMA loads into the stage ring
//     (full/empty mbarriers); an MMA warp issues a tile's 2*KS MMAs once the 8 compute
//     warps have written its A and B (a_full) and commits to mma_bar; the accumulator
//     is double-buffered, so the compute warps drain tile j-1 while the MMAs of tile j
//     run.  (A 1-CTA/SM variant with 16 compute warps and double-buffered A measured
//     slower: more per-warp overhead, one pipeline per SM.)
#pragma once
#include "tc_common.cuh"

namespace stapk {

constexpr int kApplyTcComputeWarps = 8;                        // 2 per TMEM lane quarter
constexpr int kApplyTcThreads = kApplyTcComputeWarps * 32 + 64;  // + producer warp + MMA warp
constexpr int kApplyTcTmemCols = 256;  // A hi [0,64) | A lo [64,128) | accumulators x 2 [128,256)
constexpr int kApplyTcSmemBudget = 112 * 1024;  // two CTAs per SM

// shared memory: B (KS k-steps x 64 rows x 32 B: rows 0-31 hi, 32-63 lo) | ns stages |
// barriers.  A stage holds the N snapshot rows of a tile (512 B
// each) and, for a unit's first tile, its S x N weights.
__host__ __device__ inline uint32_t apply_tc_b_bytes(int KS) { return (uint32_t)KS * 2048u; }
// a stage: NP = 8*ceil(N/8) snapshot rows of 512 B (rows N..NP-1 stay zero: the A loads
// need no bounds test) then the unit's S x N weights
__host__ __device__ inline uint32_t apply_tc_stage_bytes(int N) {
  return (uint32_t)((N + 7) & ~7) * 512u + (uint32_t)N * 16u * 8u;
}
__host__ inline int apply_tc_stages(int N) {
  const int KS = (N + 7) / 8;
  const int ns = (int)((kApplyTcSmemBudget - apply_tc_b_bytes(KS) - 512) / apply_tc_stage_bytes(N));
  return ns < 2 ? 2 : ns > 8 ? 8 : ns;
}
__host__ inline size_t apply_tc_smem_bytes(int N) {
  const int KS = (N + 7) / 8;
  const size_t need = (size_t)apply_tc_b_bytes(KS) + (size_t)apply_tc_stages(N) * apply_tc_stage_bytes(N) + 512;
  return need < 80 * 1024 ? 80 * 1024 : need;  // >= 80 KB caps residency at 2 CTAs per SM (TMEM)
}
__host__ inline bool apply_tc_supported(int N, int S, int K) { return S == 16 && K % 64 == 0 && N >= 1 && N <= 64; }

// Two CTAs per SM, each walking units u = blockIdx.x, +gridDim.x, ...; a unit is K/64
// tiles of 64 cells.  Tile j of the CTA uses stage j % ns and accumulator j & 1.  Per
// k-step two MMAs: Ahi x [Bhi; Blo] (N = 64) into
// accumulator columns [0,64) and Alo x Bhi (N = 32) into [0,32); the epilogue adds
// column c and c + 32.
// REMOTE: Y stores go through st_y (multicast / peer copies); the plain instantiation
// compiles to ordinary stores only.
template <int KS, bool REMOTE>
__global__ void __launch_bounds__(kApplyTcThreads, 2)
    apply_tc_kernel(const __grid_constant__ CUtensorMap cube_map, KParams p, const float2* __restrict__ wts,
                    float2* __restrict__ out, int units, int ns) {
  constexpr int S = 16, NP = 8 * KS;
  constexpr int kCompute = kApplyTcComputeWarps * 32;
  extern __shared__ __align__(128) unsigned char smem[];  // no-swizzle descriptors need 16 B
  const int N = p.N, K = p.K, C = p.C, D = p.D, R = p.R;
  unsigned char* bbuf = smem;
  unsigned char* stage0 = smem + apply_tc_b_bytes(KS);
  const uint32_t stage_bytes = apply_tc_stage_bytes(N);
  uint64_t* full = reinterpret_cast<uint64_t*>(stage0 + (size_t)ns * stage_bytes);  // stage loaded
  uint64_t* empty = full + ns;                                                      // stage read
  uint64_t* a_full = empty + ns;   // A (TMEM) and B (smem) of the tile written
  uint64_t* mma_bar = a_full + 1;  // the tile's MMAs done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mma_bar + 1);
  // warp index and TMEM base broadcast from lane 0: provably warp-uniform, so the compiler keeps
  // them (and the TMEM addresses derived from them) in uniform registers
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kApplyTcTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCompute);
    }
    mbar_init(a_full, kCompute);
    mbar_init(mma_bar, 1);
    fence_mbar_init();
  }
  for (int s = 0; s < ns; ++s)  // snapshot rows N..NP-1 of every stage: zero, never written by TMA
    for (int i = tid; i < (NP - N) * 128; i += blockDim.x)
      reinterpret_cast<float*>(stage0 + (size_t)s * stage_bytes + (size_t)N * 512)[i] = 0.f;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const int MT = K / 64;
  const int G = gridDim.x;
  const int my_units = (int)blockIdx.x < units ? (units - (int)blockIdx.x + G - 1) / G : 0;
  const int ntiles = my_units * MT;
  const int Gq = G / p.B, Gr = G - Gq * p.B;

  struct Tile {
    int u, mt, b, nd, q;  // unit, 64-cell tile in the unit, block, (cube, bin) row, unit count
  };
  Tile t;  // this warp's current tile
  t.u = (int)blockIdx.x;
  t.mt = 0;
  t.nd = t.u / p.B;
  t.b = t.u - t.nd * p.B;
  t.q = 0;
  auto advance = [&](Tile& x) {  // this CTA's next tile: next 64 cells, else unit u + G
    if (++x.mt == MT) {
      x.mt = 0;
      x.u += G;
      ++x.q;
      x.nd += Gq;
      x.b += Gr;
      if (x.b >= p.B) {
        x.b -= p.B;
        ++x.nd;
      }
    }
  };

  if (warp == kApplyTcComputeWarps) {
    // ---- producer (one thread): per tile, TMA-load the N snapshot rows -- per lag t one
    // {64 cells, C channels} box of the cube viewed as [batch*nbins*C rows][2R floats] --
    // and, for a unit's first tile, bulk-copy its S x N weights; all complete on full[s]
    if (lane == 0) {
      const uint32_t wbytes = (uint32_t)(S * N * 8);
      int s = 0;
      uint32_t ph = 0;
      for (int j = 0; j < ntiles; ++j) {
        if (j >= ns) mbar_wait(&empty[s], ph ^ 1u);  // the compute warps have read tile j - ns
        const int n = t.nd / p.dop_count, d = p.dop_begin + (t.nd - n * p.dop_count);
        const int base = local_bin(p, d - p.h);  // local row of bin d-h; the window wraps mod D
        unsigned char* dst = stage0 + (size_t)s * stage_bytes;
        mbar_arrive_expect_tx(&full[s], (uint32_t)N * 512u + (t.mt == 0 ? wbytes : 0u));
        if (t.mt == 0) bulk_g2s(dst + (size_t)NP * 512, wts + (long long)t.u * S * N, wbytes, &full[s]);
        const int x = 2 * (t.b * K + t.mt * 64), y0 = n * p.nbins * C;
        for (int tt = 0; tt < p.T; ++tt) {
          int lb = base + tt;
          lb -= lb >= D ? D : 0;
          tma_load_2d(dst + (size_t)tt * C * 512, &cube_map, x, y0 + lb * C, &full[s]);
        }
        advance(t);
        if (++s == ns) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
  } else if (warp == kApplyTcComputeWarps + 1) {
    // ---- MMA issuer (one thread)
    if (lane == 0) {
      const uint32_t id64 = umma_idesc_tf32(128, 64), id32 = umma_idesc_tf32(128, 32);
      for (int j = 0; j < ntiles; ++j) {
        mbar_wait(a_full, (uint32_t)j & 1u);
        tc_fence_after();
        const uint32_t bb = smem_u32(bbuf);
        const uint32_t acc = tmem + 128 + 64 * (j & 1), ahi = tmem, alo = tmem + 64;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const uint64_t bd = umma_desc(bb + ks * 2048, 128, 256);
          umma_tf32_ts(acc, ahi + 8 * ks, bd, id64, ks > 0);  // Ahi x [Bhi; Blo]
          umma_tf32_ts(acc, alo + 8 * ks, bd, id32, 1);       // Alo x Bhi (rows 0-31 of B)
        }
        umma_commit(mma_bar);
      }
    }
  } else {
    // ---- compute warps: warp w owns TMEM lane quarter q4 = w % 4 (rows m = 32 q4 + lane),
    // k-steps hq, hq + 2, ... (hq = w / 4) of A, and steering k in [8hq, 8hq + 8)
    const int q4 = warp & 3, hq = warp >> 2;
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    const int m = q4 * 32 + lane, jj = m >> 1, part = m & 1;
    constexpr int KH = (KS + 1) / 2;  // k-steps per warp (at most)

    // weights (in the stage) -> B buffer: K-major rows nn = lo*32 + part*16 + k, column i
    auto stage_b = [&](const float2* wg, unsigned char* bb) {
      const int i3 = lane & 3, k7 = lane >> 2;  // a warp stores 128 contiguous bytes
      for (int g = warp; g < 2 * (NP / 4); g += kApplyTcComputeWarps) {
        const int i = (g >> 1) * 4 + i3, k = (g & 1) * 8 + k7;
        const float2 w = i < N ? wg[k * N + i] : make_float2(0.f, 0.f);
#pragma unroll
        for (int pp = 0; pp < 2; ++pp) {
          const int nn = pp * S + k;
          const float x = pp ? w.y : w.x;
          const uint32_t off =
              (uint32_t)(i >> 3) * 2048u + (nn >> 3) * 256 + ((i >> 2) & 1) * 128 + (nn & 7) * 16 + (i & 3) * 4;
          *reinterpret_cast<float*>(bb + off) = x;                                // hi (truncated by the MMA)
          *reinterpret_cast<float*>(bb + off + 4 * 256) = x - tf32_trunc(x);     // lo, row nn + 32
        }
      }
    };
    // accumulator of tile x (parity par) -> Y[k][cell] for k in [8hq, 8hq+8)
    auto epilogue = [&](const Tile& x, int par) {
      float a[8], b[8], c[8], d[8];
      const uint32_t acc = tmem + lane_base + 128 + 64 * par + 8 * hq;
      tmem_ld8x4(acc, acc + S, acc + 32, acc + 32 + S, a, b, c, d);
      float* yp = reinterpret_cast<float*>(out + (long long)x.nd * S * R + (long long)(8 * hq) * R +
                                           (long long)x.b * K + x.mt * 64 + jj) + part;
      const float sg = part ? -1.f : 1.f;  // Re: own + partner; Im: own - partner
      float yv[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float re = a[k] + c[k];                                  // Out[m][k]
        const float o = __shfl_xor_sync(0xffffffffu, b[k] + d[k], 1);  // partner row's Out[.][S+k]
        yv[k] = fmaf(sg, o, re);
      }
      if constexpr (REMOTE) {
#pragma unroll
        for (int k = 0; k < 8; ++k) st_y(yp + (long long)k * 2 * R, yv[k], p);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) yp[(long long)k * 2 * R] = yv[k];
      }
    };

    Tile prev = t;
    int s = 0;
    uint32_t ph = 0;
    for (int j = 0; j < ntiles; ++j) {
      const float* zs = reinterpret_cast<const float*>(stage0 + (size_t)s * stage_bytes) + m;
      mbar_wait(&full[s], ph);
      float z[KH][8];
#pragma unroll
      for (int kh = 0; kh < KH; ++kh) {
        const float* zk = zs + (hq + 2 * kh) * 8 * 128;  // rows 8ks .. 8ks+7 (padding rows are zero)
#pragma unroll
        for (int e = 0; e < 8; ++e) z[kh][e] = (hq + 2 * kh < KS) ? zk[e * 128] : 0.f;
      }
      if (j >= 1) {  // MMA(j-1) done: A, B and accumulator (j-1) & 1 are ready
        mbar_wait(mma_bar, (uint32_t)(j - 1) & 1u);
        tc_fence_after();
      }
      if (t.mt == 0) {
        stage_b(reinterpret_cast<const float2*>(stage0 + (size_t)s * stage_bytes + (size_t)NP * 512), bbuf);
        fence_proxy_async();  // generic-proxy B stores -> visible to the tensor core
      }
      // A: row m, k-steps hq + 2kh: hi at column 8ks, lo at 64 + 8ks
#pragma unroll
      for (int kh = 0; kh < KH; ++kh) {
        const int ks = hq + 2 * kh;
        if (ks < KS) {
          float l[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) l[e] = z[kh][e] - tf32_trunc(z[kh][e]);
          tmem_st8(tmem + lane_base + 8 * ks, z[kh]);  // hi: the tensor core truncates to TF32
          tmem_st8(tmem + lane_base + 64 + 8 * ks, l);
        }
      }
      // release the stage only after its values have been used (an mbarrier arrive does
      // not wait for this thread's outstanding shared loads)
      mbar_arrive(&empty[s]);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      mbar_arrive(a_full);
      if (j >= 1) {  // drain tile j-1 while MMA(j) runs
        epilogue(prev, (j - 1) & 1);
        tc_fence_before();
      }
      prev = t;
      advance(t);
      if (++s == ns) {
        s = 0;
        ph ^= 1u;
      }
    }
    if (ntiles > 0) {
      const int jl = ntiles - 1;
      mbar_wait(mma_bar, (uint32_t)jl & 1u);
      tc_fence_after();
      epilogue(prev, jl & 1);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kApplyTcTmemCols));
}

}  // namespace stapk

// apply_run.cuh -- K3 on the tcgen05 tensor cores in Doppler-run order: every snapshot row is
// staged and split into TF32 hi/lo ONCE per run of consecutive Doppler bins, instead of once
// per output bin whose window contains it (T times; apply_tc.cuh).
//
// Method: Y[d][k][r] = w_{d,b(r),k}^H z_{d,r} (reading c-12; "applying the
// weights to every range cell of the datacube"), per tile of 64 range cells of a unit (d, b),
// as the real GEMM of apply_tc.cuh (rows m = 2*cell + part, columns [Re w; Im w] hi then lo,
// 3xTF32 = Ahi Bhi + Ahi Blo + Alo Bhi, FP32 accumulation in tensor memory).  The reduction
// runs over the window: k-step t of unit d is Doppler bin d - h + t, its C channels padded to
// the 8 elements of a TF32 k-step (weights of the padding are zero).
//
// Run order.  A CTA walks chunks of PCH consecutive bins of one "line" (cube n, block b, 64-cell
// tile mt).  Along a chunk, consecutive units share T-1 of their T window bins, so each bin is
// TMA-loaded (one {64 cells, C channels} box) and split into hi/lo once, into a ring of 8 TMEM
// slots (16 columns each: hi, lo); unit d's MMAs read slots (d - h + t) mod 8 directly -- the
// A operand is never copied again.  A chunk starts with T-1 warm-up bins.
//
// Pipeline (two persistent CTAs per SM, 256 TMEM columns each: ring [0,128) | accumulators
// x 2 [128,256)): a producer warp TMA-loads one bin per stage (plus, for a unit, its S x N
// weights) into a ring of shared-memory stages; four compute warps split the bin into its TMEM
// slot, all eight stage the unit's B (weights, canonical K-major, double-buffered by unit
// parity); an MMA warp issues the unit's 2T MMAs; the accumulator is double-buffered, so the
// eight compute warps drain unit j-1 while unit j's MMAs run.
#pragma once
#include "tc_common.cuh"

namespace stapk {

constexpr int kApplyRunCompute = 8;                         // compute warps (2 per TMEM lane quarter)
constexpr int kApplyRunThreads = kApplyRunCompute * 32 + 64;  // + producer warp + MMA warp
constexpr int kApplyRunTmemCols = 256;                       // ring of 8 bins x (hi 8 | lo 8) | acc x 2
constexpr int kApplyRunSlots = 8;
constexpr int kApplyRunSmemBudget = 112 * 1024;  // two CTAs per SM

// the shapes it runs: S = 16, K % 64 == 0, C <= 8, T <= 7 (ring of 8 bins covers a window + 1)
__host__ inline bool apply_run_supported(int C, int T, int S, int K) {
  return S == 16 && K % 64 == 0 && C >= 1 && C <= 8 && T >= 1 && T <= kApplyRunSlots - 1;
}
// B per unit: T k-steps x 64 rows x 32 B
__host__ __device__ inline uint32_t apply_run_b_bytes(int T) { return (uint32_t)T * 2048u; }
// a stage: one bin (C rows of 512 B) then the unit's S x N weights
__host__ __device__ inline uint32_t apply_run_stage_bytes(int C, int N) {
  return (((uint32_t)C * 512u + (uint32_t)N * 16u * 8u) + 127u) & ~127u;
}
__host__ inline int apply_run_stages(int C, int T, int N) {
  const int ns = (int)((kApplyRunSmemBudget - 2 * apply_run_b_bytes(T) - 1024) / apply_run_stage_bytes(C, N));
  return ns < 2 ? 2 : ns > 12 ? 12 : ns;
}
__host__ inline size_t apply_run_smem_bytes(int C, int T, int N) {
  const size_t need = 2 * (size_t)apply_run_b_bytes(T) + (size_t)apply_run_stages(C, T, N) * apply_run_stage_bytes(C, N) + 1024;
  return need < 80 * 1024 ? 80 * 1024 : need;  // >= 80 KB caps residency at 2 CTAs per SM (TMEM)
}

// The chunk schedule shared by the three roles: chunk q of the CTA -> (line, first bin, bins).
struct RunSched {
  int lines_per_n;  // B * MT
  int cpl;          // chunks per line = ceil(Dl / PCH)
  int pch;          // bins per chunk
  int nchunks;      // batch * B * MT * cpl
};

template <bool REMOTE>
__global__ void __launch_bounds__(kApplyRunThreads, 2)
    apply_run_kernel(const __grid_constant__ CUtensorMap cube_map, KParams p, const float2* __restrict__ wts,
                     float2* __restrict__ out, RunSched sc, int ns) {
  constexpr int S = 16;
  constexpr int kCompute = kApplyRunCompute * 32;
  extern __shared__ __align__(128) unsigned char smem[];  // no-swizzle descriptors need 16 B
  const int N = p.N, K = p.K, C = p.C, T = p.T, D = p.D, R = p.R, Dl = p.dop_count;
  const int MT = K / 64;
  const uint32_t bbytes = apply_run_b_bytes(T);
  unsigned char* bbuf = smem;  // [2][T][64 rows x 32 B] by unit parity
  unsigned char* stage0 = smem + 2 * bbytes;
  const uint32_t stage_bytes = apply_run_stage_bytes(C, N);
  uint64_t* full = reinterpret_cast<uint64_t*>(stage0 + (size_t)ns * stage_bytes);  // stage loaded
  uint64_t* empty = full + ns;                                                      // stage consumed
  uint64_t* a_full = empty + ns;   // [2] by unit parity: A slots and B of the unit written
  uint64_t* mma_bar = a_full + 2;  // [2] by unit parity: the unit's MMAs done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mma_bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kApplyRunTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCompute);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&a_full[b], kCompute);
      mbar_init(&mma_bar[b], 1);
    }
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // chunk q of this CTA (q = blockIdx.x + i * gridDim.x) -> n, b, mt, first owned bin index dl0, bins
  struct Chunk {
    int n, b, mt, dl0, nb;
  };
  auto chunk = [&](int q) {
    Chunk c;
    const int line = q / sc.cpl, part = q - line * sc.cpl;
    c.n = line / sc.lines_per_n;
    const int lb = line - c.n * sc.lines_per_n;
    c.b = lb / MT;
    c.mt = lb - c.b * MT;
    c.dl0 = part * sc.pch;
    c.nb = min(sc.pch, Dl - c.dl0);
    return c;
  };

  if (warp == kApplyRunCompute) {
    // ---- producer (one thread): per chunk T-1 warm-up bins, then per unit one bin + weights
    if (lane == 0) {
      const uint32_t wbytes = (uint32_t)(S * N * 8);
      int s = 0;
      uint32_t ph = 0;
      int e = 0;  // stage events
      for (int q = blockIdx.x; q < sc.nchunks; q += gridDim.x) {
        const Chunk c = chunk(q);
        const int y0 = c.n * p.nbins * C, x = 2 * (c.b * K + c.mt * 64);
        const int wbase = local_bin(p, p.dop_begin + c.dl0 - p.h);  // local row of the chunk's first window bin
        for (int i = 0; i < c.nb + T - 1; ++i, ++e) {
          if (e >= ns) mbar_wait(&empty[s], ph ^ 1u);
          unsigned char* dst = stage0 + (size_t)s * stage_bytes;
          const bool unit = i >= T - 1;
          mbar_arrive_expect_tx(&full[s], (uint32_t)C * 512u + (unit ? wbytes : 0u));
          int lb = wbase + i;
          while (lb >= D) lb -= D;
          tma_load_2d(dst, &cube_map, x, y0 + lb * C, &full[s]);
          if (unit) {
            const long long u = ((long long)c.n * Dl + c.dl0 + (i - (T - 1))) * p.B + c.b;
            bulk_g2s(dst + (size_t)C * 512, wts + u * S * N, wbytes, &full[s]);
          }
          if (++s == ns) {
            s = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == kApplyRunCompute + 1) {
    // ---- MMA issuer (one thread): per unit, 2T MMAs over its window's ring slots
    if (lane == 0) {
      const uint32_t id64 = umma_idesc_tf32(128, 64), id32 = umma_idesc_tf32(128, 32);
      int j = 0;       // units
      uint32_t cnt = 0;  // bins entered into the ring
      for (int q = blockIdx.x; q < sc.nchunks; q += gridDim.x) {
        const Chunk c = chunk(q);
        cnt += (uint32_t)(T - 1);  // warm-up bins
        for (int r = 0; r < c.nb; ++r, ++j) {
          const uint32_t first = cnt + 1 - (uint32_t)T;  // ring counter of the window's first bin
          ++cnt;
          mbar_wait(&a_full[j & 1], (uint32_t)(j >> 1) & 1u);
          tc_fence_after();
          const uint32_t bb = smem_u32(bbuf) + (uint32_t)(j & 1) * bbytes;
          const uint32_t acc = tmem + 128 + 64 * (j & 1);
          for (int t = 0; t < T; ++t) {
            const uint32_t slot = (first + (uint32_t)t) & (kApplyRunSlots - 1);
            const uint32_t ahi = tmem + 16 * slot, alo = ahi + 8;
            const uint64_t bd = umma_desc(bb + t * 2048, 128, 256);
            umma_tf32_ts(acc, ahi, bd, id64, t > 0);  // Ahi x [Bhi; Blo]
            umma_tf32_ts(acc, alo, bd, id32, 1);      // Alo x Bhi (rows 0-31 of B)
          }
          umma_commit(&mma_bar[j & 1]);
        }
      }
    }
  } else {
    // ---- compute warps: warp w owns TMEM lane quarter q4 = w % 4 (rows m = 32 q4 + lane);
    // warps 0-3 split the bins, all eight stage B; the epilogue's steering half is hq = w / 4
    const int q4 = warp & 3, hq = warp >> 2;
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    const int m = q4 * 32 + lane, jj = m >> 1, part = m & 1;

    // weights (in the stage, [S][N]) -> B buffer: K-major rows nn = lo*32 + part*16 + k,
    // column i' = 8t + c (snapshot element t*C + c; zero for c >= C)
    auto stage_b = [&](const float2* wg, unsigned char* bb) {
      const int i3 = lane & 3, k7 = lane >> 2;  // a warp stores 128 contiguous bytes
      for (int g = warp; g < 4 * T; g += kApplyRunCompute) {  // 2 groups of 4 columns x 2 k-halves per k-step
        const int ip = (g >> 1) * 4 + i3, k = (g & 1) * 8 + k7;  // ip = 8t + c
        const int t = ip >> 3, cc = ip & 7;
        const float2 w = cc < C ? wg[k * N + t * C + cc] : make_float2(0.f, 0.f);
#pragma unroll
        for (int pp = 0; pp < 2; ++pp) {
          const int nn = pp * S + k;
          const float xw = pp ? w.y : w.x;
          const uint32_t off =
              (uint32_t)(ip >> 3) * 2048u + (nn >> 3) * 256 + ((ip >> 2) & 1) * 128 + (nn & 7) * 16 + (ip & 3) * 4;
          *reinterpret_cast<float*>(bb + off) = xw;                              // hi (truncated by the MMA)
          *reinterpret_cast<float*>(bb + off + 4 * 256) = xw - tf32_trunc(xw);  // lo, row nn + 32
        }
      }
    };
    // accumulator of unit x (parity par) -> Y[k][cell] for k in [8hq, 8hq+8)
    auto epilogue = [&](long long ybase, int par) {
      float a[8], b[8], c[8], d[8];
      const uint32_t acc = tmem + lane_base + 128 + 64 * par + 8 * hq;
      tmem_ld8x4(acc, acc + S, acc + 32, acc + 32 + S, a, b, c, d);
      float* yp = reinterpret_cast<float*>(out + ybase + (long long)(8 * hq) * R + jj) + part;
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

    int s = 0;
    uint32_t ph = 0;
    int j = 0;  // units
    uint32_t cnt = 0;  // bins entered into the ring
    long long yprev = 0;
    for (int q = blockIdx.x; q < sc.nchunks; q += gridDim.x) {
      const Chunk c = chunk(q);
      for (int i = 0; i < c.nb + T - 1; ++i) {
        const bool unit = i >= T - 1;
        // the TMEM slot this bin overwrites, the B buffer and the accumulator of unit j must be
        // free: at a chunk's first bin every earlier unit's MMAs (the new window overlaps the last
        // ones'), inside a chunk unit j-2's (the last reader of the slot 8 bins back, T <= 7)
        if (i == 0 && j >= 1) {
          mbar_wait(&mma_bar[(j - 1) & 1], (uint32_t)((j - 1) >> 1) & 1u);
          if (j >= 2) mbar_wait(&mma_bar[j & 1], (uint32_t)((j - 2) >> 1) & 1u);
          tc_fence_after();
        } else if (unit && i > T - 1 && j >= 2) {
          mbar_wait(&mma_bar[j & 1], (uint32_t)((j - 2) >> 1) & 1u);
          tc_fence_after();
        }
        mbar_wait(&full[s], ph);
        const float* zs = reinterpret_cast<const float*>(stage0 + (size_t)s * stage_bytes) + m;
        if (hq == 0) {  // split the bin into its ring slot: hi at 16 slot, lo at 16 slot + 8
          float z[8], l[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) z[e] = e < C ? zs[e * 128] : 0.f;
#pragma unroll
          for (int e = 0; e < 8; ++e) l[e] = z[e] - tf32_trunc(z[e]);
          const uint32_t slot = cnt & (kApplyRunSlots - 1);
          tmem_st8(tmem + lane_base + 16 * slot, z);  // hi: the tensor core truncates to TF32
          tmem_st8(tmem + lane_base + 16 * slot + 8, l);
        }
        ++cnt;
        if (unit) {
          stage_b(reinterpret_cast<const float2*>(stage0 + (size_t)s * stage_bytes + (size_t)C * 512),
                  bbuf + (size_t)(j & 1) * bbytes);
          fence_proxy_async();  // generic-proxy B stores -> visible to the tensor core
        }
        // release the stage only after its values have been used (an mbarrier arrive does not
        // wait for this thread's outstanding shared loads)
        mbar_arrive(&empty[s]);
        if (++s == ns) {
          s = 0;
          ph ^= 1u;
        }
        if (!unit) continue;
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(&a_full[j & 1]);
        if (j >= 1) {  // drain unit j-1 while unit j's MMAs run
          mbar_wait(&mma_bar[(j - 1) & 1], (uint32_t)((j - 1) >> 1) & 1u);
          tc_fence_after();
          epilogue(yprev, (j - 1) & 1);
          tc_fence_before();
        }
        const int dl = c.dl0 + (i - (T - 1));
        yprev = (((long long)c.n * Dl + dl) * S) * R + (long long)c.b * K + c.mt * 64;
        ++j;
      }
    }
    if (j > 0) {
      const int jl = j - 1;
      mbar_wait(&mma_bar[jl & 1], (uint32_t)(jl >> 1) & 1u);
      tc_fence_after();
      epilogue(yprev, jl & 1);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kApplyRunTmemCols));
}

// the chunk length: balance chunks over the CTAs against the T-1 warm-up bins per chunk
__host__ inline RunSched apply_run_schedule(int batch, int B, int MT, int Dl, int T, int ctas) {
  RunSched best{};
  double best_cost = 1e30;
  const int cands[] = {16, 24, 32, 48, 64, 96, 128, 192, 256};
  for (int pch : cands) {
    RunSched s;
    s.lines_per_n = B * MT;
    s.pch = pch;
    s.cpl = (Dl + pch - 1) / pch;
    s.nchunks = batch * B * MT * s.cpl;
    // bins per CTA on the busiest CTA: chunks rounded up over the CTAs, each pch + T - 1 bins
    const double rounds = (double)((s.nchunks + ctas - 1) / ctas);
    const double cost = rounds * (pch + T - 1) + 0.0 * pch;
    if (cost < best_cost) {
      best_cost = cost;
      best = s;
    }
    if (pch >= Dl) break;
  }
  return best;
}

}  // namespace stapk

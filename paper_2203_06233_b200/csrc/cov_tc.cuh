// cov_tc.cuh -- K1 on the 5th-generation tensor cores (tcgen05.mma kind::tf32, 3xTF32).
//
// Method (include/stap.h; readings c-4..c-7 -- the paper gives the STAP kernel
// only as a figure): R_hat_d =
// (1/K) sum_r z_r z_r^H over the K cells of a training block, z_r[t*C + c] =
// X[d-h+t][c][r]; R_d = R_hat_d + delta_d I, delta_d = lambda tr(R_hat_d) / N.
//
// Every entry of R_hat_d is an entry of the Gram matrix of the cube rows (bin w,
// channel c) over the block's cells: R_hat_d[(t1,c1),(t2,c2)] = G[(d-h+t1,c1),
// (d-h+t2,c2)] / K with G[m][n] = sum_r x_m[r] conj(x_n[r]).  A CTA tile takes MB =
// 128/C consecutive bins (M = 128 Gram rows), computes the 128 x 128 Gram block of
// those rows with themselves, and emits R_d for the OB = MB - T + 1 bins whose
// windows lie inside the tile (adjacent tiles overlap by T-1 bins).  As real GEMMs
// over the cells k of a 16-cell chunk (re / im de-interleaved):
//   Re G = Re_m . Re_n + Im_m . Im_n,   Im G = Im_m . Re_n - Re_m . Im_n
// each product in 3xTF32 (x = hi + lo, hi = x rounded to TF32, lo = x - hi; the
// tensor core truncates lo to TF32), so 12 MMAs (M = N = 128, K = 8) per 8 cells,
// the negated ones via the instruction descriptor's negate-A bit.
//
// Data movement: a producer warp TMA-loads each chunk of the tile (one box {32
// floats, MB*C rows} of the cube viewed as [batch*nbins*C rows][2R floats], 128-byte
// swizzled so that a thread reading its own row is bank-conflict free) into a ring of
// 2-4 stages (as many as the shared memory holds: 3 at large, 4 at medium); the rare tiles whose bins wrap around the cube's edge read rows from global.
// Four compute warps (thread m = Gram row m = TMEM lane m) read their row, split it
// and write (a) the A operand into their TMEM lane (the "TS" form: A never touches
// shared memory again) and (b) the B operand planes (Re hi, Im hi, Re lo, Im lo,
// canonical K-major no-swizzle layout) into shared memory.  An MMA warp issues the
// 24 MMAs of a chunk into the two accumulators (Re G at TMEM columns [128,256), Im G
// at [256,384)); A and B are double-buffered per chunk.  After the tile's last chunk
// the compute warps copy the band of their Gram row (the T*C columns from the
// diagonal on) and its conjugate mirror into a shared buffer of Gram rows, then write
// every R_d of the tile row by row, coalesced, from contiguous pieces of those rows --
// R_d is exactly Hermitian (mirrored entries are bit-exact conjugates), diagonal real.
#pragma once
#include "tc_common.cuh"

namespace stapk {

#ifdef COVTC_PROF  // dev builds only: per-phase cycle counters of compute thread 0
__device__ unsigned long long g_covtc_prof[8];  // [6] = tiles; [7] = band copy without the delta part
#define COVTC_T(v) const long long v = clock64()
#define COVTC_ADD(i, x) \
  if (tid == 0) atomicAdd(&g_covtc_prof[i], (unsigned long long)(x))
#else
#define COVTC_T(v)
#define COVTC_ADD(i, x)
#endif

constexpr int kCovTcCompute = 4;  // compute warps: TMEM lanes 0..127
constexpr int kCovTcWriter = 8;   // writer warps: R_d assembly and stores, overlapped with the next tile
constexpr int kCovTcThreads = (kCovTcCompute + kCovTcWriter) * 32 + 64;  // + producer warp + MMA warp
constexpr uint32_t kCovTcRawBytes = 128u * 128u;        // a chunk: 128 rows x 32 floats (16 cells)
constexpr uint32_t kCovTcPlaneBytes = 128u * 16u * 4u;  // a B plane: 128 rows x 16 cells
constexpr uint32_t kCovTcBBytes = 4u * kCovTcPlaneBytes;  // Re hi | Im hi | Re lo | Im lo
constexpr int kCovTcTmemCols = 512;  // A x 2 buffers [0,128) | Re G [128,256) | Im G [256,384)

struct CovTcGeom {
  int MB;   // bins per tile (MB * C <= 128 Gram rows)
  int OB;   // output bins per tile = MB - T + 1
  int ntd;  // tiles along the owned Doppler range
  int RS;   // row stride (float2) of the Gram band buffer: >= N with RS - 1 odd (conflict-free)
  int NS;   // stages of the TMA chunk ring: as many (2..4) as fit the shared memory
};
__host__ inline CovTcGeom cov_tc_geom(int C, int T, int N, int dop_count) {
  CovTcGeom g;
  g.MB = 128 / C;
  g.OB = g.MB - T + 1;
  g.ntd = g.OB > 0 ? (dop_count + g.OB - 1) / g.OB : 0;
  g.RS = (N & 1) ? N + 1 : N;  // RS - 1 odd: band writes and mirrored reads of consecutive lanes
  g.NS = 2;                     // set by the plan (cov_tc_smem decides what fits)
  return g;
}
// Where it is used: the 128 x 128 Gram tile is worth it only when the window (N = T*C
// rows) covers a good part of it -- measured on B200: large (N = 56) 613 vs 1095 us,
// medium (N = 30) 542 vs 807 us per step, small (N = 12) 640 vs 260 us (SIMT kept).
__host__ inline bool cov_tc_supported(int C, int T, int N, int K) {
  return C >= 1 && C <= 8 && 128 / C >= T && K % 16 == 0 && N >= 24 && N <= 64;
}
struct CovTcSmem {
  size_t raw, bpl, rbuf, delta, bar, total;
};
__host__ __device__ inline CovTcSmem cov_tc_smem(int N, int RS, int OB, int NS) {
  CovTcSmem s;
  s.raw = 0;                                           // stages (1024-aligned for the swizzle)
  s.bpl = s.raw + (size_t)NS * kCovTcRawBytes;         // B planes x 2
  s.rbuf = s.bpl + 2 * (size_t)kCovTcBBytes;           // Gram band x 2 [128][RS]
  s.delta = s.rbuf + 2 * (size_t)128 * RS * 8;         // delta x 2 [OB]
  s.bar = s.delta + 2 * (((size_t)OB * 4 + 15) & ~(size_t)15);
  s.total = s.bar + (2 * NS + 8) * 8 + 16 + 1024;  // + alignment slack
  return s;
}

__global__ void __launch_bounds__(kCovTcThreads, 1)
    cov_tc_kernel(const __grid_constant__ CUtensorMap map_sw, KParams p, const float2* __restrict__ cube,
                  float2* __restrict__ cov, int ntiles, CovTcGeom g) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const int C = p.C, T = p.T, N = p.N, K = p.K;
  const CovTcSmem L = cov_tc_smem(N, g.RS, g.OB, g.NS);
  const int NS = g.NS;
  unsigned char* raw = smem + L.raw;
  unsigned char* bpl = smem + L.bpl;
  float2* gband0 = reinterpret_cast<float2*>(smem + L.rbuf);  // [2][128][RS]: band G[m][m+k] / K
  float* delta0 = reinterpret_cast<float*>(smem + L.delta);    // [2][OB4]
  const int OB4 = ((g.OB + 3) & ~3);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar);  // [stages]
  uint64_t* empty = full + NS;                        // [stages]
  uint64_t* a_full = empty + NS;                      // [2] by chunk parity
  uint64_t* mma_done = a_full + 2;                              // [2] by chunk parity
  uint64_t* gb_full = mma_done + 2;   // [2] by tile parity: band written (compute -> writers)
  uint64_t* gb_empty = gb_full + 2;   // [2] by tile parity: band consumed (writers -> compute)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gb_empty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int kCompute = kCovTcCompute * 32;
  constexpr uint32_t ACC_RE = 128, ACC_IM = 256;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kCovTcTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCompute);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&a_full[b], kCompute);
      mbar_init(&mma_done[b], 1);
      mbar_init(&gb_full[b], kCompute);
      mbar_init(&gb_empty[b], kCovTcWriter * 32);
    }
    fence_mbar_init();
  }
  // rows a tile leaves unloaded (MB*C < 128) must hold finite values
  for (uint32_t i = tid; i < NS * kCovTcRawBytes / 16; i += blockDim.x)
    reinterpret_cast<float4*>(raw)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nch = K / 16;

  struct Tile {
    int n, b, d0, OBt, MBt, lr0;
    bool wrap;
  };
  auto decode = [&](int tt) {
    Tile t;
    t.b = tt % p.B;
    const int r = tt / p.B;
    const int td = r % g.ntd;
    t.n = r / g.ntd;
    t.d0 = p.dop_begin + td * g.OB;
    t.OBt = min(g.OB, p.dop_count - td * g.OB);
    t.MBt = t.OBt + T - 1;
    t.lr0 = local_bin(p, t.d0 - p.h);
    t.wrap = t.lr0 + t.MBt > p.D;
#ifdef COVTC_FORCE_BIN
    t.wrap = true;
#endif
    return t;
  };

  if (warp >= kCovTcCompute + 2) {
    // ---- writer warps: per tile, delta of its output bins and every R_d, from the band
    // R_d[i][l] = G[m0+i][m0+l] / K: for l >= i the band of row m0+i, for l < i the
    // conjugate of the band entry of row m0+l (one load either way, no branch; mirrored
    // entries are bit-exact conjugates); the loading on the (real) diagonal.  Rows by
    // warp, two columns per lane, 16-byte coalesced stores.
    const int wt = tid - (kCovTcCompute + 2) * 32, ww = wt >> 5;
    const int l0 = 2 * lane;
    int j = 0;
    for (int tt = blockIdx.x; tt < ntiles; tt += gridDim.x, ++j) {
      const Tile t = decode(tt);
      const int pb = j & 1;
      const float2* gb = gband0 + (size_t)pb * 128 * g.RS;
      float* dls = delta0 + pb * OB4;
      mbar_wait(&gb_full[pb], (uint32_t)(j >> 1) & 1u);
      if (wt < t.OBt) {  // delta of output bin wt: lambda * sum_i Rhat[i][i] (ascending i) / N
        float tr = 0.f;
        for (int i = 0; i < N; ++i) tr += gb[(wt * C + i) * g.RS].x;
        dls[wt] = p.lam * tr / (float)N;
      }
      asm volatile("bar.sync 2, %0;" ::"r"(kCovTcWriter * 32) : "memory");
      auto rget = [&](int m0, int i, int l, float dlt) {
        const bool up = l >= i;
        const float2 u = gb[(up ? (m0 + i) : (m0 + l)) * g.RS + (up ? l - i : i - l)];
        return l == i ? make_float2(u.x + dlt, 0.f) : (up ? u : make_float2(u.x, -u.y));
      };
      for (int di = 0; di < t.OBt; ++di) {
        const int m0 = di * C;
        const float dlt = dls[di];
        const int dl = t.d0 - p.dop_begin + di;
        float2* o = cov + (((long long)t.n * p.dop_count + dl) * p.B + t.b) * (long long)N * N;
        if ((N & 1) == 0) {
#pragma unroll 4
          for (int i = ww; i < N; i += kCovTcWriter) {
            if (l0 < N) {
              const float2 v0 = rget(m0, i, l0, dlt), v1 = rget(m0, i, l0 + 1, dlt);
              *reinterpret_cast<float4*>(o + i * N + l0) = make_float4(v0.x, v0.y, v1.x, v1.y);
            }
          }
        } else {
          for (int i = ww; i < N; i += kCovTcWriter)
            for (int l = lane; l < N; l += 32) o[i * N + l] = rget(m0, i, l, dlt);
        }
      }
      mbar_arrive(&gb_empty[pb]);  // (all reads of this band and of dls precede: stores consumed them)
    }
  } else if (warp == kCovTcCompute) {
    // ---- producer (one thread): chunk ch of a tile = cells [b*K + 16ch, +16) of its rows
    if (lane == 0) {
      int s = 0, cc = 0;
      uint32_t ph = 0;
      for (int tt = blockIdx.x; tt < ntiles; tt += gridDim.x) {
        const Tile t = decode(tt);
        const int y0 = t.n * p.nbins * C;
        for (int ch = 0; ch < nch; ++ch, ++cc) {
          if (cc >= NS) mbar_wait(&empty[s], ph ^ 1u);
          unsigned char* dst = raw + (size_t)s * kCovTcRawBytes;
          const int x = 2 * (t.b * K + 16 * ch);
          if (!t.wrap) {
            mbar_arrive_expect_tx(&full[s], (uint32_t)(g.MB * C) * 128u);
            tma_load_2d(dst, &map_sw, x, y0 + t.lr0 * C, &full[s]);
          } else {
            mbar_arrive(&full[s]);  // wrapped tile: the compute warps read their rows from global memory
          }
          if (++s == NS) {
            s = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == kCovTcCompute + 1) {
    // ---- MMA issuer (one thread): 24 MMAs per chunk
    if (lane == 0) {
      const uint32_t id = umma_idesc_tf32(128, 128), idn = umma_idesc_tf32(128, 128, true);
      int cc = 0;
      for (int tt = blockIdx.x; tt < ntiles; tt += gridDim.x) {
        for (int ch = 0; ch < nch; ++ch, ++cc) {
          const int pb = cc & 1;
          mbar_wait(&a_full[pb], (uint32_t)(cc >> 1) & 1u);
          tc_fence_after();
          const uint32_t ab = tmem + 64 * pb, bb = smem_u32(bpl + (size_t)pb * kCovTcBBytes);
          const uint32_t re = tmem + ACC_RE, im = tmem + ACC_IM;
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const uint32_t ko = ks * 4096;
            const uint64_t bRH = umma_desc(bb + ko, 128, 256), bIH = umma_desc(bb + kCovTcPlaneBytes + ko, 128, 256);
            const uint64_t bRL = umma_desc(bb + 2 * kCovTcPlaneBytes + ko, 128, 256);
            const uint64_t bIL = umma_desc(bb + 3 * kCovTcPlaneBytes + ko, 128, 256);
            const uint32_t aRH = ab + 8 * ks, aIH = ab + 16 + 8 * ks, aRL = ab + 32 + 8 * ks, aIL = ab + 48 + 8 * ks;
            const uint32_t acc0 = (ch > 0 || ks > 0) ? 1u : 0u;
            umma_tf32_ts(re, aRH, bRH, id, acc0);  // Re G += Re_m Re_n + Im_m Im_n
            umma_tf32_ts(re, aRH, bRL, id, 1);
            umma_tf32_ts(re, aRL, bRH, id, 1);
            umma_tf32_ts(re, aIH, bIH, id, 1);
            umma_tf32_ts(re, aIH, bIL, id, 1);
            umma_tf32_ts(re, aIL, bIH, id, 1);
            umma_tf32_ts(im, aIH, bRH, id, acc0);  // Im G += Im_m Re_n - Re_m Im_n
            umma_tf32_ts(im, aIH, bRL, id, 1);
            umma_tf32_ts(im, aIL, bRH, id, 1);
            umma_tf32_ts(im, aRH, bIH, idn, 1);
            umma_tf32_ts(im, aRH, bIL, idn, 1);
            umma_tf32_ts(im, aRL, bIH, idn, 1);
          }
          umma_commit(&mma_done[pb]);
        }
      }
    }
  } else {
    // ---- compute warps: thread m = Gram row m = TMEM lane m
    const int m = tid;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const float invK = 1.0f / (float)K;
    int s = 0, cc = 0, tj = 0;
    uint32_t ph = 0;
    for (int tt = blockIdx.x; tt < ntiles; tt += gridDim.x) {
      const Tile t = decode(tt);
      COVTC_T(q0);
      for (int ch = 0; ch < nch; ++ch, ++cc) {
        const int pb = cc & 1;
        COVTC_T(w0);
        mbar_wait(&full[s], ph);
        COVTC_T(w1);
        COVTC_ADD(0, w1 - w0);
        // row m: 8 x 16 B = cells 0..15 as (re, im) pairs, 128-byte swizzled in the stage; a
        // tile whose bins wrap around the cube edge reads its rows from global memory
        const unsigned char* rrow = raw + (size_t)s * kCovTcRawBytes + (size_t)m * 128;
        const int wm = m / C, cm = m - wm * C;
        const float4* grow = reinterpret_cast<const float4*>(
            cube + ((long long)t.n * p.nbins + local_bin(p, t.d0 - p.h + min(wm, t.MBt - 1))) * C * p.R +
            (long long)cm * p.R + (long long)t.b * K + 16 * ch);
        float re[16], imv[16];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 q = t.wrap ? __ldg(grow + j) : *reinterpret_cast<const float4*>(rrow + (j ^ (m & 7)) * 16);
          re[2 * j] = q.x;
          imv[2 * j] = q.y;
          re[2 * j + 1] = q.z;
          imv[2 * j + 1] = q.w;
        }
        float rh[16], ih[16], rl[16], il[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          rh[e] = tf32_hi(re[e]);
          rl[e] = re[e] - rh[e];
          ih[e] = tf32_hi(imv[e]);
          il[e] = imv[e] - ih[e];
        }
        COVTC_T(w2);
        if (cc >= 2) {  // MMAs of chunk cc-2 done: A buffer pb and B planes pb are free
          mbar_wait(&mma_done[pb], (uint32_t)((cc - 2) >> 1) & 1u);
          tc_fence_after();
        }
        COVTC_T(w3);
        COVTC_ADD(1, w3 - w2);
        const uint32_t ab = tmem + lane_base + 64 * pb;
        tmem_st8(ab, rh);
        tmem_st8(ab + 8, rh + 8);
        tmem_st8(ab + 16, ih);
        tmem_st8(ab + 24, ih + 8);
        tmem_st8(ab + 32, rl);
        tmem_st8(ab + 40, rl + 8);
        tmem_st8(ab + 48, il);
        tmem_st8(ab + 56, il + 8);
        // release the stage only here: the tcgen05.st above consume (as asm operands) values
        // derived from every loaded element, so the shared loads have completed.  An
        // mbarrier arrive does not wait for outstanding loads, and the compiler may sink
        // plain arithmetic below an arrive, so an earlier release let the next TMA
        // overwrite a row mid-read (seen as run-to-run differences in one Gram row/column)
        mbar_arrive(&empty[s]);
        // B planes, K-major core matrices: (row m, cell k) at (k/8)*4096 + (m/8)*256 +
        // ((k/4)%2)*128 + (m%8)*16 + (k%4)*4 -- four cells per 16-byte store
        unsigned char* bp = bpl + (size_t)pb * kCovTcBBytes + (m >> 3) * 256 + (m & 7) * 16;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t o = (q >> 1) * 4096 + (q & 1) * 128;
          *reinterpret_cast<float4*>(bp + o) = make_float4(rh[4 * q], rh[4 * q + 1], rh[4 * q + 2], rh[4 * q + 3]);
          *reinterpret_cast<float4*>(bp + kCovTcPlaneBytes + o) =
              make_float4(ih[4 * q], ih[4 * q + 1], ih[4 * q + 2], ih[4 * q + 3]);
          *reinterpret_cast<float4*>(bp + 2 * kCovTcPlaneBytes + o) =
              make_float4(rl[4 * q], rl[4 * q + 1], rl[4 * q + 2], rl[4 * q + 3]);
          *reinterpret_cast<float4*>(bp + 3 * kCovTcPlaneBytes + o) =
              make_float4(il[4 * q], il[4 * q + 1], il[4 * q + 2], il[4 * q + 3]);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        fence_proxy_async();  // generic-proxy B stores -> visible to the tensor core
        tc_fence_before();
        mbar_arrive(&a_full[pb]);
        if (++s == NS) {
          s = 0;
          ph ^= 1u;
        }
      }

      // ---- G of this tile is complete once the last chunk's MMAs are: thread m copies the
      // band of its Gram row, G[m][m .. end of bin(m)+T-1] / K, to gband[tile parity][m][n - m]
      // (own row, conflict-free; the warp reads the union of its lanes' columns from TMEM)
      // and hands it to the writer warps, then goes on to the next tile.
      const int last = cc - 1;
      COVTC_T(q1);
      COVTC_ADD(2, q1 - q0);
      mbar_wait(&mma_done[last & 1], (uint32_t)(last >> 1) & 1u);
      tc_fence_after();
      COVTC_T(q2);
      COVTC_ADD(3, q2 - q1);
      {
        const int pbt = tj & 1;
        if (tj >= 2) mbar_wait(&gb_empty[pbt], (uint32_t)((tj - 2) >> 1) & 1u);  // writers done with tile tj-2
        float2* grow = gband0 + (size_t)pbt * 128 * g.RS + m * g.RS;
        const int nend = (m / C + T) * C;  // one past the last band column of row m
        const int cbeg = warp * 32, cend = min(cbeg + 31 + N, 128);
        for (int c0 = cbeg; c0 < cend; c0 += 16) {  // 16 columns (Re, Im) per TMEM round trip
          float vr[16], vi[16];
          tmem_ld8x4(tmem + lane_base + ACC_RE + c0, tmem + lane_base + ACC_IM + c0,
                     tmem + lane_base + ACC_RE + c0 + 8, tmem + lane_base + ACC_IM + c0 + 8,
                     *reinterpret_cast<float(*)[8]>(vr), *reinterpret_cast<float(*)[8]>(vi),
                     *reinterpret_cast<float(*)[8]>(vr + 8), *reinterpret_cast<float(*)[8]>(vi + 8));
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int n = c0 + e, k = n - m;
            if (k >= 0 && n < nend) grow[k] = make_float2(vr[e] * invK, vi[e] * invK);
          }
        }
        tc_fence_before();
        mbar_arrive(&gb_full[pbt]);
      }
      COVTC_T(q3);
      COVTC_ADD(4, q3 - q2);
      ++tj;
      COVTC_T(q4);
      COVTC_ADD(5, q4 - q3);
      COVTC_ADD(6, 1);
      tc_fence_before();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCovTcTmemCols));
}

}  // namespace stapk

// cov.cuh -- K1: loaded covariance of every owned unit (d, b).
//
// Method (include/stap.h; readings c-2..c-7): for unit (d, b) the
// snapshot rows are z[t*C + c][j] = X[(d-h+t) mod D][c][bK + j] and
//   Rhat[i][l] = (1/K) sum_j z[i][j] conj(z[l][j]),  R = Rhat + (lambda tr(Rhat)/N) I.
//
// B200 design -- Doppler-lag block sharing: the (t, t')
// C x C block of R_d is P(a, a') = (1/K) sum_j x_a[.][j] x_a'[.][j]^H with
// a = d-h+t, a' = d-h+t', so a CTA that owns a run of P consecutive bins of one
// training block computes every lag block (w, w+l), l < T, of its window of
// W = P+T-1 bins ONCE and assembles the P matrices from them: T*W - T(T-1)/2
// blocks instead of P*T(T+1)/2.  Each block's sum runs over j in ascending
// order no matter which CTA computes it, so the result is bitwise independent
// of P, of the run alignment and of the Doppler shard.
//
// Staging: the window is streamed through shared memory in chunks of KC range
// cells with 1-D bulk async copies (TMA engine, one copy per (bin, channel)
// row, completing on an mbarrier), double-buffered so the copy of chunk c+2
// overlaps the math on chunk c+1.  Tile layout [w][c][KC+2] plus 2 complex per
// bin: the 16-byte row pad and bin pad put the rows two threads of a block and
// four consecutive bins read on distinct 16-byte bank groups.  Two threads own
// one lag block for even C >= 4 (TI = C/2 rows x C columns each, adjacent
// lanes, so the column operand is a broadcast), one thread otherwise; complex
// accumulators in registers, float4 (2 cells) loads along j.
#pragma once
#include "common.cuh"

namespace stapk {

__host__ __device__ inline int cov_blocks(int T, int W) { return T * W - T * (T - 1) / 2; }
// staged lag-block stride (complex): C*C + 1 so the same element of consecutive blocks
// falls on different banks (the HERK writes and the R assembly reads are conflict-free)
__host__ __device__ inline int blk_stride(int C) { return C * C + 1; }
// threads per lag block: C=4 -> 4 (one row each), other even C >= 6 -> 2 (C/2 rows), odd C -> 1
__host__ __device__ constexpr int cov_tpb(int C) { return C == 4 ? 4 : ((C >= 6 && (C & 1) == 0) ? 2 : 1); }
__host__ __device__ inline int tile_rs(int KC) { return KC + 2; }                             // row stride (complex)
__host__ __device__ inline int tile_bs(int C, int KC) { return C * (KC + 2) + 2; }            // bin stride (complex)
// largest even divisor of K that is <= 32
__host__ __device__ inline int cov_kc(int K) {
  for (int kc = K < 32 ? K : 32; kc >= 2; kc -= 2)
    if (K % kc == 0) return kc;
  return 2;
}

struct CovLayout {
  int KC, nchunks, nbuf;
  size_t tile_bytes, body, total;
};
__host__ __device__ inline CovLayout cov_layout(int C, int T, int K, int P) {
  CovLayout L;
  L.KC = cov_kc(K);
  L.nchunks = K / L.KC;
  L.nbuf = L.nchunks > 1 ? 2 : 1;
  L.tile_bytes = (((size_t)(P + T - 1) * tile_bs(C, L.KC) * 8) + 127) & ~(size_t)127;
  size_t body = L.nbuf * L.tile_bytes;
  const size_t blk = (size_t)cov_blocks(T, P + T - 1) * blk_stride(C) * 8;
  if (blk > body) body = blk;
  L.body = (body + 127) & ~(size_t)127;
  L.total = L.body + 16 /*2 mbarriers*/ + (size_t)P * 4 /*delta*/ + 16;
  return L;
}
__host__ inline size_t cov_smem_bytes(int C, int T, int K, int P) { return cov_layout(C, T, K, P).total; }

// Issue the bulk copies of cells [j0, j0+KC) of the W-bin window (global bins
// d0-h .. d0-h+W-1, wrapped) of training block b of cube n into tile; the
// mbarrier `bar` completes when all bytes have landed.  Every thread of the CTA
// issues its share of the (bin, channel) row copies (one copy per thread for
// typical windows), so the copies start together; one thread must have posted
// the expected byte count on `bar` (window_chunk_bytes) before, behind a barrier.
__host__ __device__ inline uint32_t window_chunk_bytes(int W, int C, int KC) { return (uint32_t)(W * C * KC * 8); }
__device__ __forceinline__ void issue_window_chunk(const KParams& p, const float2* __restrict__ cube, int n, int b,
                                                   int d0, int W, int C, int j0, int KC, float2* tile,
                                                   uint64_t* bar) {
  const int rs = tile_rs(KC), bs = tile_bs(C, KC);
  const float2* cb = cube + (long long)n * p.cube_stride + (long long)b * p.K + j0;
  for (int q = threadIdx.x; q < W * C; q += blockDim.x) {
    const int w = q / C, c = q - w * C;
    const int lb = local_bin(p, d0 - p.h + w);
    bulk_g2s(tile + w * bs + c * rs, cb + ((long long)lb * C + c) * p.R, (uint32_t)(KC * 8), bar);
  }
}

// Lag-major block enumeration: block index t -> (w, l), block (w, w+l), w < W - l.
__device__ __forceinline__ void lag_block_of(int t, int T, int W, int& w, int& l) {
  l = 0;
  w = t;
  while (l < T && w >= W - l) {
    w -= W - l;
    ++l;
  }
}
__host__ __device__ inline int lag_block_index(int w, int l, int W) { return l * W - l * (l - 1) / 2 + w; }

// acc[u][c2] += sum_{j < KC} xa[u][j] conj(xb[c2][j]), j ascending (fixed order);
// xa = TI rows (stride rs), xb = C rows (stride rs).
template <int C, int TI>
__device__ __forceinline__ void herk_chunk(const float2* xa, const float2* xb, int rs, int KC,
                                           float2 (&acc)[TI][C]) {
#pragma unroll(C >= 8 ? 1 : 2)
  for (int j = 0; j < KC; j += 2) {
    float4 a[TI];
#pragma unroll
    for (int u = 0; u < TI; ++u) a[u] = *reinterpret_cast<const float4*>(xa + u * rs + j);
#pragma unroll
    for (int c2 = 0; c2 < C; ++c2) {
      const float4 bb = *reinterpret_cast<const float4*>(xb + c2 * rs + j);
#pragma unroll
      for (int u = 0; u < TI; ++u) {
        cmac_conj(acc[u][c2], make_float2(a[u].x, a[u].y), make_float2(bb.x, bb.y));
        cmac_conj(acc[u][c2], make_float2(a[u].z, a[u].w), make_float2(bb.z, bb.w));
      }
    }
  }
}

// Element (i, l) of Rhat for bin p of a run from the scaled lag blocks blk[nblk][C][C]:
// upper (t_i, c_i) <= (t_l, c_l) read directly, lower = conj of the mirrored upper.
__device__ __forceinline__ float2 rhat_from_blocks(const float2* blk, int C, int W, int pr, int i, int col) {
  const int ti = i / C, ci = i - ti * C, tl = col / C, cl = col - tl * C;
  if (ti < tl || (ti == tl && ci <= cl)) {
    return blk[lag_block_index(pr + ti, tl - ti, W) * blk_stride(C) + ci * C + cl];
  }
  const float2 u = blk[lag_block_index(pr + tl, ti - tl, W) * blk_stride(C) + cl * C + ci];
  return make_float2(u.x, -u.y);
}

// delta of bin pr: lambda * sum_{i ascending} Re Rhat[i][i] / N  (lag-0 block of bin w is index w).
__device__ __forceinline__ float delta_from_blocks(const float2* blk, int C, int T, int N, float lam, int pr) {
  float tr = 0.f;
  for (int t = 0; t < T; ++t)
    for (int c = 0; c < C; ++c) tr += blk[(pr + t) * blk_stride(C) + c * C + c].x;
  return lam * tr / (float)N;
}

// The lag-block HERK of one CTA over all K cells, streaming chunks through
// `tiles` (nbuf buffers) with mbarriers bar[0..1]; on return (after a CTA
// barrier) the scaled blocks are in blk[nblk][C][C] (which may alias tiles).
template <int C>
__device__ __forceinline__ void cta_lag_blocks(const KParams& p, const float2* __restrict__ cube, int n, int b,
                                               int d0, int W, const CovLayout& L, unsigned char* tiles,
                                               uint64_t* bar, float2* blk) {
  constexpr int TPB = cov_tpb(C);
  constexpr int TI = C / TPB;
  const int tid = threadIdx.x;
  const int T = p.T;
  const int nblk = cov_blocks(T, W);
  const int KC = L.KC, rs = tile_rs(KC), bs = tile_bs(C, KC);
  const uint32_t cbytes = window_chunk_bytes(W, C, KC);
  if (tid == 0) {
    mbar_arrive_expect_tx(bar, cbytes);
    if (L.nchunks > 1) mbar_arrive_expect_tx(bar + 1, cbytes);
  }
  __syncthreads();
  issue_window_chunk(p, cube, n, b, d0, W, C, 0, KC, reinterpret_cast<float2*>(tiles), bar);
  if (L.nchunks > 1)
    issue_window_chunk(p, cube, n, b, d0, W, C, KC, KC, reinterpret_cast<float2*>(tiles + L.tile_bytes), bar + 1);
  const int bi = tid / TPB, hf = tid - bi * TPB;
  int w, l;
  lag_block_of(bi, T, W, w, l);
  const bool active = bi < nblk;
  float2 acc[TI][C];
#pragma unroll
  for (int u = 0; u < TI; ++u)
#pragma unroll
    for (int c2 = 0; c2 < C; ++c2) acc[u][c2] = make_float2(0.f, 0.f);
  for (int ch = 0; ch < L.nchunks; ++ch) {
    const int buf = ch & 1;
    const float2* tile = reinterpret_cast<const float2*>(tiles + buf * L.tile_bytes);
    mbar_wait(bar + buf, (ch >> 1) & 1);
    if (active) herk_chunk<C, TI>(tile + w * bs + hf * TI * rs, tile + (w + l) * bs, rs, KC, acc);
    if (tid == 0 && ch + 2 < L.nchunks) mbar_arrive_expect_tx(bar + buf, cbytes);  // next phase of this buffer
    __syncthreads();  // every thread is done with this buffer
    if (ch + 2 < L.nchunks)
      issue_window_chunk(p, cube, n, b, d0, W, C, (ch + 2) * KC, KC,
                         reinterpret_cast<float2*>(tiles + buf * L.tile_bytes), bar + buf);
  }
  const float invK = 1.0f / (float)p.K;
  if (active) {
#pragma unroll
    for (int u = 0; u < TI; ++u)
#pragma unroll
      for (int c2 = 0; c2 < C; ++c2)
        blk[bi * blk_stride(C) + (hf * TI + u) * C + c2] = make_float2(acc[u][c2].x * invK, acc[u][c2].y * invK);
  }
  __syncthreads();
}

template <int C>
__global__ void __launch_bounds__(256, ((C & 1) && C >= 5) ? 1 : 2) cov_kernel(KParams p, const float2* __restrict__ cube,
                                                   float2* __restrict__ cov, int P) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int run = blockIdx.x, b = blockIdx.y, n = blockIdx.z;
  const int T = p.T, N = p.N;
  const int dl0 = run * P;                  // first owned (local) bin of this run
  const int Prun = min(P, p.dop_count - dl0);
  const int d0 = p.dop_begin + dl0;         // its global index
  const int W = Prun + T - 1;
  const CovLayout L = cov_layout(C, T, p.K, P);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.body);
  float* delta_s = reinterpret_cast<float*>(smem + L.body + 16);
  float2* blk = reinterpret_cast<float2*>(smem);  // aliases the tiles after the HERK

  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_mbar_init();
  }
  __syncthreads();
  cta_lag_blocks<C>(p, cube, n, b, d0, W, L, smem, bar, blk);

  if (tid < Prun) delta_s[tid] = delta_from_blocks(blk, C, T, N, p.lam, tid);
  __syncthreads();

  // Assemble R_d for each bin of the run (both triangles; lower = conj of upper).
  // R_d is T x T tiles of C x C; tile (ti, tl) is lag block (pr + min, |tl - ti|),
  // conjugate-transposed below the diagonal.  A lane owns one element pair
  // (ci, 2cp..2cp+1) of a tile (fixed for the whole loop); a warp covers
  // 32 / (C * ceil(C/2)) tiles per pass, so the index math is per tile, not per element.
  constexpr int CP = (C + 1) / 2;  // element pairs per tile row
  constexpr int LPT = C * CP;      // lanes per tile
  constexpr int TPW = 32 / LPT;    // tiles per warp pass
  const long long NN = (long long)N * N;
  float2* out = cov + (((long long)n * p.dop_count + dl0) * p.B + b) * NN;
  const long long ostride = (long long)p.B * NN;  // between consecutive bins
  const int lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int slot = lane / LPT, e = lane - slot * LPT;
  const int ci = e / CP, c0 = 2 * (e - (e / CP) * CP);
  const bool two = c0 + 1 < C;
  const int TT = T * T, ntiles = Prun * TT, bsd = blk_stride(C);
  for (int t0 = warp * TPW; t0 < ntiles; t0 += nwarps * TPW) {
    const int t = t0 + slot;
    if (slot >= TPW || t >= ntiles) continue;
    const int pr = t / TT, rem = t - pr * TT;
    const int ti = rem / T, tl = rem - ti * T;
    float2 v0, v1;
    if (ti < tl) {
      const float2* s = blk + lag_block_index(pr + ti, tl - ti, W) * bsd + ci * C + c0;
      v0 = s[0];
      v1 = two ? s[1] : make_float2(0.f, 0.f);
    } else if (ti > tl) {
      const float2* s = blk + lag_block_index(pr + tl, ti - tl, W) * bsd + c0 * C + ci;
      const float2 u0 = s[0], u1 = two ? s[C] : make_float2(0.f, 0.f);
      v0 = make_float2(u0.x, -u0.y);
      v1 = make_float2(u1.x, -u1.y);
    } else {  // diagonal tile: upper from the block, lower mirrored, loading on the diagonal
      const float2* s = blk + lag_block_index(pr + ti, 0, W) * bsd;
      const float dl = delta_s[pr];
      float2 x[2];
#pragma unroll
      for (int q2 = 0; q2 < 2; ++q2) {
        const int cl = c0 + q2;
        if (q2 == 1 && !two) {
          x[q2] = make_float2(0.f, 0.f);
          continue;
        }
        if (ci < cl) {
          x[q2] = s[ci * C + cl];
        } else if (ci > cl) {
          const float2 u = s[cl * C + ci];
          x[q2] = make_float2(u.x, -u.y);
        } else {
          x[q2] = make_float2(s[ci * C + ci].x + dl, 0.f);
        }
      }
      v0 = x[0];
      v1 = x[1];
    }
    float2* o = out + pr * ostride + (long long)(ti * C + ci) * N + tl * C + c0;
    if ((C & 1) == 0) {
      *reinterpret_cast<float4*>(o) = make_float4(v0.x, v0.y, v1.x, v1.y);  // N even: 16-byte aligned
    } else {
      o[0] = v0;
      if (two) o[1] = v1;
    }
  }
}

}  // namespace stapk

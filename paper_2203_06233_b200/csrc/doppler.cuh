// doppler.cuh -- K0, the Doppler front end (reading c-19):
//   X[d][c][r] = sum_{p < D} w[p] x[p][c][r] exp(-2 pi i p d / D)
// the per-row taper and FFT along the pulse axis that turn raw pulses into the datacube
// (Table 2 "fft_2D,axis=1"; Fig. 7 text).
//
// B200 design: HBM-bound (one read and one write of the cube; the FFT's 5 D log2 D flops
// per column are far below the ridge).  A CTA takes RC consecutive range cells of one
// channel of one cube -- every pulse row of that tile is one contiguous RC*8-byte
// piece, so loads and stores are coalesced -- keeps the D x RC tile in shared memory,
// and runs an in-place radix-2 decimation-in-time FFT on every column: the taper is
// applied at the load, which also scatters rows to bit-reversed positions; the log2(D)
// butterfly stages follow two at a time (radix-4 passes), threads over (butterfly, cell) with the cell index fastest
// so a warp touches consecutive words of one or two rows (bank-conflict free).
// Twiddles exp(-2 pi i k / D), k < D/2, come from sincospif into shared memory once per
// CTA.  D must be a power of two (2 .. 8192).
#pragma once
#include "common.cuh"

namespace stapk {

constexpr int kDopplerThreads = 256;
constexpr size_t kDopplerTileBytes = 48 * 1024;  // four CTAs per SM

// cells per CTA: the largest power of two <= 64 that divides R and keeps D*RC*8 + the
// twiddles within kDopplerTileBytes
__host__ inline int doppler_rc(int D, int R) {
  int rc = 64;
  while (rc > 1 && ((size_t)D * rc * 8 + (size_t)D / 2 * 8 > kDopplerTileBytes || R % rc)) rc >>= 1;
  return rc;
}
__host__ inline size_t doppler_smem(int D, int rc) { return (size_t)D * rc * 8 + (size_t)(D / 2) * 8; }

__device__ __forceinline__ int bitrev(int x, int bits) { return (int)(__brev((unsigned)x) >> (32 - bits)); }

__global__ void __launch_bounds__(kDopplerThreads, 4)
    doppler_kernel(const float2* __restrict__ raw, const float* __restrict__ window, float2* __restrict__ out,
                   int D, int logD, int C, int R, int lrc) {
  const int rc = 1 << lrc, jm = rc - 1;
  extern __shared__ __align__(16) float2 dsm[];
  float2* tile = dsm;           // [D][rc]
  float2* tw = dsm + D * rc;    // [D/2]
  const int r0 = blockIdx.x * rc, c = blockIdx.y, n = blockIdx.z;
  const long long plane = (long long)C * R;
  const float2* src = raw + (long long)n * D * plane + (long long)c * R + r0;
  float2* dst = out + (long long)n * D * plane + (long long)c * R + r0;
  const int tid = threadIdx.x;
  for (int k = tid; k < D / 2; k += blockDim.x) {
    float s, co;
    sincospif(-2.0f * (float)k / (float)D, &s, &co);
    tw[k] = make_float2(co, s);
  }
  // load + taper, rows to bit-reversed positions
#pragma unroll 4
  for (int idx = tid; idx < D * rc; idx += blockDim.x) {
    const int p = idx >> lrc, j = idx & jm;
    const float2 v = __ldg(src + (long long)p * plane + j);
    const float w = __ldg(window + p);
    tile[(bitrev(p, logD) << lrc) + j] = make_float2(v.x * w, v.y * w);
  }
  __syncthreads();
  // radix-2 DIT stages (span 2h, twiddle exp(-2 pi i pos / 2h) = tw[pos * D / 2h]), two at a
  // time: a thread takes the 4 elements i0 + {0, h, 2h, 3h} of a span-4h group through
  // stage s (pairs (i0,i1), (i2,i3), twiddle W_2h^pos) and stage s+1 (pairs (i0,i2) with
  // W_4h^pos, (i1,i3) with W_4h^(pos+h)) in registers -- the same operations as two
  // radix-2 passes, half the shared-memory passes and barriers
  auto bfly = [](float2& a, float2& u, float2 t) {
    const float2 bu = make_float2(fmaf(u.x, t.x, -u.y * t.y), fmaf(u.x, t.y, u.y * t.x));
    u = make_float2(a.x - bu.x, a.y - bu.y);
    a = make_float2(a.x + bu.x, a.y + bu.y);
  };
  int s = 0;
  for (; s + 1 < logD; s += 2) {
    const int h = 1 << s, t1 = D >> (s + 1), t2 = D >> (s + 2);
#pragma unroll 2
    for (int b = tid; b < (D / 4) * rc; b += blockDim.x) {
      const int k = b >> lrc, j = b & jm;
      const int pos = k & (h - 1), i0 = ((k >> s) << (s + 2)) + pos;
      float2 x0 = tile[(i0 << lrc) + j], x1 = tile[((i0 + h) << lrc) + j];
      float2 x2 = tile[((i0 + 2 * h) << lrc) + j], x3 = tile[((i0 + 3 * h) << lrc) + j];
      const float2 w1 = tw[pos * t1];
      bfly(x0, x1, w1);
      bfly(x2, x3, w1);
      bfly(x0, x2, tw[pos * t2]);
      bfly(x1, x3, tw[(pos + h) * t2]);
      tile[(i0 << lrc) + j] = x0;
      tile[((i0 + h) << lrc) + j] = x1;
      tile[((i0 + 2 * h) << lrc) + j] = x2;
      tile[((i0 + 3 * h) << lrc) + j] = x3;
    }
    __syncthreads();
  }
  if (s < logD) {  // odd log2 D: one last radix-2 stage
    const int h = 1 << s, tstride = D >> (s + 1);
    for (int b = tid; b < (D / 2) * rc; b += blockDim.x) {
      const int k = b >> lrc, j = b & jm;
      const int pos = k & (h - 1), i0 = ((k >> s) << (s + 1)) + pos;
      float2 a = tile[(i0 << lrc) + j], u = tile[((i0 + h) << lrc) + j];
      bfly(a, u, tw[pos * tstride]);
      tile[(i0 << lrc) + j] = a;
      tile[((i0 + h) << lrc) + j] = u;
    }
    __syncthreads();
  }
#pragma unroll 4
  for (int idx = tid; idx < D * rc; idx += blockDim.x) {
    const int d = idx >> lrc, j = idx & jm;
    dst[(long long)d * plane + j] = tile[idx];
  }
}

// ---------------------------------------------------------------------------------------
// K0b, the register path for 16 <= D <= 1024: D = L1*L2 (L1, L2 <= 32), one Cooley-Tukey
// split (n = L2*m + q, d = k1 + L1*k2):
//   A[q][k1] = sum_m w[L2 m + q] x[L2 m + q] W_L1^(m k1)      (L1-point DFT, registers)
//   B[q][k1] = A[q][k1] * W_D^(q k1)                            (twiddle, to shared memory)
//   X[k1 + L1 k2] = sum_q B[q][k1] W_L2^(q k2)                  (L2-point DFT, registers)
// -- the same sum as the windowed DFT, regrouped.  Step 1 reads its L1 pulses straight from
// HBM (a warp covers 32/rc pulse rows of rc*8 contiguous bytes), step 2 writes its L2 bins
// straight to HBM; shared memory is crossed once (write + read) instead of log2(D)/2 times,
// which is what bounded K0 (measured: 12 tile traversals per 2 HBM crossings at D = 1024).
// In-register DFTs are radix-2 DIT with compile-time indices (bit reversal is renaming);
// W_32^k comes from a literal table in constant memory.

__constant__ float2 c_w32[16] = {
    {1.000000000e+00f, 0.000000000e+00f},   {9.807852804e-01f, -1.950903220e-01f},
    {9.238795325e-01f, -3.826834324e-01f},  {8.314696123e-01f, -5.555702330e-01f},
    {7.071067812e-01f, -7.071067812e-01f},  {5.555702330e-01f, -8.314696123e-01f},
    {3.826834324e-01f, -9.238795325e-01f},  {1.950903220e-01f, -9.807852804e-01f},
    {0.000000000e+00f, -1.000000000e+00f},  {-1.950903220e-01f, -9.807852804e-01f},
    {-3.826834324e-01f, -9.238795325e-01f}, {-5.555702330e-01f, -8.314696123e-01f},
    {-7.071067812e-01f, -7.071067812e-01f}, {-8.314696123e-01f, -5.555702330e-01f},
    {-9.238795325e-01f, -3.826834324e-01f}, {-9.807852804e-01f, -1.950903220e-01f}};

template <int L>
__host__ __device__ constexpr int brev_c(int i) {
  int r = 0;
  for (int b = 1; b < L; b <<= 1) r = (r << 1) | ((i & b) ? 1 : 0);
  return r;
}

// in-place L-point DFT (exp(-2 pi i n k / L)) of v, natural order in and out
template <int L>
__device__ __forceinline__ void dft_reg(float2 (&v)[L]) {
  float2 a[L];
#pragma unroll
  for (int i = 0; i < L; ++i) a[brev_c<L>(i)] = v[i];
#pragma unroll
  for (int h = 1; h < L; h <<= 1) {
#pragma unroll
    for (int g = 0; g < L; g += 2 * h) {
#pragma unroll
      for (int pos = 0; pos < h; ++pos) {
        const float2 y = a[g + pos + h];
        float2 t;
        if (pos == 0) {
          t = y;
        } else if (2 * pos == h) {  // W_2h^(h/2) = -i
          t = make_float2(y.y, -y.x);
        } else {
          const float2 w = c_w32[pos * (16 / h)];  // W_2h^pos = W_32^(pos*32/2h)
          t = make_float2(fmaf(y.x, w.x, -y.y * w.y), fmaf(y.x, w.y, y.y * w.x));
        }
        const float2 x = a[g + pos];
        a[g + pos] = make_float2(x.x + t.x, x.y + t.y);
        a[g + pos + h] = make_float2(x.x - t.x, x.y - t.y);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < L; ++i) v[i] = a[i];
}

#ifndef STAP_DOPPLER2_MAX_SMEM
#define STAP_DOPPLER2_MAX_SMEM (80 * 1024)
#endif
constexpr size_t kDoppler2MaxSmem = STAP_DOPPLER2_MAX_SMEM;  // rc = 16 up to D = 512, 8 at D = 1024

// shared bytes: B tile [L1][L2*rc + pad] + twiddles W_D^n (n < D)
__host__ inline int doppler2_pad(int rc) { return rc < 16 ? rc : 0; }
__host__ inline size_t doppler2_smem(int L1, int L2, int rc) {
  return ((size_t)L1 * (L2 * rc + doppler2_pad(rc)) + (size_t)L1 * L2) * 8;
}

// CTAs per SM: 4 for L1 <= 16 (<= 64 registers, no spill), 2 for L1 = 32 (its 32 complex
// values per thread need ~128 registers; forcing 3 spills).  Measured at D = 256: 2 -> 4
// CTAs/SM took the HBM fraction from 0.67 to 0.96.
template <int L1, int L2>
__global__ void __launch_bounds__(kDopplerThreads, (L1 <= 16 ? 4 : 2))
    doppler2_kernel(const float2* __restrict__ raw, const float* __restrict__ window, float2* __restrict__ out,
                    int C, int R, int lrc, int pad) {
  constexpr int D = L1 * L2;
  const int rc = 1 << lrc, jm = rc - 1;
  const int ld = L2 * rc + pad;  // row stride of the B tile (pad: rc < 16 spreads step-2 rows over banks)
  extern __shared__ __align__(16) float2 dsm[];
  float2* tile = dsm;          // [L1][ld]: B[q][k1] at tile[k1*ld + q*rc + j]
  float2* tw = dsm + L1 * ld;  // [D]
  const int r0 = blockIdx.x * rc, c = blockIdx.y, n = blockIdx.z;
  const long long plane = (long long)C * R;
  const float2* src = raw + (long long)n * D * plane + (long long)c * R + r0;
  float2* dst = out + (long long)n * D * plane + (long long)c * R + r0;
  const int tid = threadIdx.x;
  for (int k = tid; k < D; k += kDopplerThreads) {
    float s, co;
    sincospif(-2.0f * (float)k / (float)D, &s, &co);
    tw[k] = make_float2(co, s);
  }
  __syncthreads();
  for (int item = tid; item < L2 * rc; item += kDopplerThreads) {
    const int q = item >> lrc, j = item & jm;
    float2 v[L1];
#pragma unroll
    for (int m = 0; m < L1; ++m) v[m] = __ldg(src + (long long)(L2 * m + q) * plane + j);
#pragma unroll
    for (int m = 0; m < L1; ++m) {
      const float w = __ldg(window + L2 * m + q);
      v[m] = make_float2(v[m].x * w, v[m].y * w);
    }
    dft_reg<L1>(v);
#pragma unroll
    for (int k1 = 0; k1 < L1; ++k1) {
      const float2 t = tw[q * k1];
      tile[k1 * ld + item] = make_float2(fmaf(v[k1].x, t.x, -v[k1].y * t.y), fmaf(v[k1].x, t.y, v[k1].y * t.x));
    }
  }
  __syncthreads();
  for (int item = tid; item < L1 * rc; item += kDopplerThreads) {
    const int k1 = item >> lrc, j = item & jm;
    float2 v[L2];
#pragma unroll
    for (int q = 0; q < L2; ++q) v[q] = tile[k1 * ld + q * rc + j];
    dft_reg<L2>(v);
#pragma unroll
    for (int k2 = 0; k2 < L2; ++k2) dst[(long long)(k1 + L1 * k2) * plane + j] = v[k2];
  }
}

}  // namespace stapk

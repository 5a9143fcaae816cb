// Harness for the solver experiments (experiments/README.md): chol_kernel (the product
// kernel, chol.cuh) against the warp-specialised variant (chol_ws.cuh) on random loaded
// covariances shaped like large (N = 56) and medium (N = 30); prints time, FP32 fraction and
// a hash / bitwise comparison of W, gamma and info.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -I paper_2203_06233_b200/csrc -o /tmp/chol_harness experiments/chol_harness.cu
// -DNO_WS drops the warp-specialised runs; -DVARS adds the variants listed under VARS (for
// chol_blk.cuh / chol_dbl.cuh: put that file first on the include path as chol.cuh).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <complex>
#include "../experiments/chol_ws.cuh"

using namespace stapk;
typedef std::complex<double> cd;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)
static unsigned long long rs = 88172645463325252ull;
static double urand() { rs ^= rs << 13; rs ^= rs >> 7; rs ^= rs << 17; return (rs >> 11) * (1.0 / 9007199254740992.0); }
static double nrand() { double u1 = urand() + 1e-300, u2 = urand(); return sqrt(-2 * log(u1)) * cos(2 * M_PI * u2); }
struct Prob { int N, S; long long units; std::vector<float2> R, st; };
Prob make(int N, int S, long long units, int distinct, int K) {
  Prob P{N, S, units, {}, {}};
  P.R.resize((size_t)units * N * N);
  std::vector<cd> Z((size_t)N * K);
  for (int m = 0; m < distinct; ++m) {
    for (auto& z : Z) z = cd(nrand(), nrand());
    for (int r = 0; r < 3; ++r) {
      std::vector<cd> a(N);
      for (auto& x : a) x = cd(nrand(), nrand());
      for (int k = 0; k < K; ++k) { cd g(nrand() * 30, nrand() * 30); for (int i = 0; i < N; ++i) Z[i * K + k] += g * a[i]; }
    }
    std::vector<cd> Rm((size_t)N * N); double tr = 0;
    for (int i = 0; i < N; ++i) for (int l = 0; l < N; ++l) {
      cd acc = 0; for (int k = 0; k < K; ++k) acc += Z[i * K + k] * std::conj(Z[l * K + k]);
      Rm[i * N + l] = acc / (double)K; if (i == l) tr += acc.real() / K;
    }
    for (int i = 0; i < N; ++i) Rm[i * N + i] += 1e-2 * tr / N;
    for (int i = 0; i < N * N; ++i) P.R[(size_t)m * N * N + i] = make_float2((float)Rm[i].real(), (float)Rm[i].imag());
  }
  for (long long u = distinct; u < units; ++u) memcpy(&P.R[(size_t)u * N * N], &P.R[(size_t)(u % distinct) * N * N], sizeof(float2) * N * N);
  // a few failing units: a negative diagonal
  P.R[(size_t)7 * N * N + 5 * N + 5].x = -1.f;
  P.st.resize((size_t)S * N);
  for (auto& x : P.st) x = make_float2((float)nrand(), (float)nrand());
  return P;
}
struct Dev { float2 *R, *st, *W; float* g; int* info; };
template <class F> float timeit(F f, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); CK(cudaDeviceSynchronize());
  cudaEventRecord(a); for (int i = 0; i < reps; ++i) f(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b); return ms / reps * 1000.f;
}
static void fetch(const Prob& P, Dev& d, std::vector<float2>& W, std::vector<float>& g, std::vector<int>& inf) {
  W.resize((size_t)P.units * P.S * P.N); g.resize(P.units * P.S); inf.resize(P.units);
  CK(cudaMemcpy(W.data(), d.W, W.size() * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(g.data(), d.g, g.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(inf.data(), d.info, inf.size() * 4, cudaMemcpyDeviceToHost));
}
static void report(const Prob& P, const char* name, float us, int regs, size_t spill, int nb) {
  double fl = (4.0 / 3 * P.N * P.N * P.N + 8.0 * P.N * P.N * P.S) * P.units;
  printf("%-36s %9.1f us  %6.2f TF/s  %.3f of 74.4  regs=%d spill=%zu blk/SM=%d\n", name, us, fl / us * 1e-6, fl / us * 1e-6 / 74.45, regs, spill, nb);
}
template <class CF, int threads, int MINB>
void run_ref(const Prob& P, Dev& d, std::vector<float2>& W, std::vector<float>& g, std::vector<int>& inf) {
  size_t smem = (threads / CF::G) * chol_shared_bytes<CF>();
  auto k = chol_kernel<CF, threads, MINB>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k);
  int nb = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, threads, smem);
  long long per = threads / CF::G, sg = (P.units + per - 1) / per;
  int grid = (int)(sg < 148LL * nb ? sg : 148LL * nb);
  CK(cudaMemset(d.W, 0xff, (size_t)P.units * P.S * P.N * 8));
  float us = timeit([&] { k<<<grid, threads, smem>>>(P.N, P.S, P.units, d.R, d.st, d.W, d.g, d.info); }, 10);
  CK(cudaGetLastError());
  report(P, "chol_kernel (ref)", us, fa.numRegs, fa.localSizeBytes, nb);
  fetch(P, d, W, g, inf);
  unsigned long long h = 1469598103934665603ull;
  const unsigned char* b = (const unsigned char*)W.data();
  for (size_t i = 0; i < W.size() * 8; ++i) h = (h ^ b[i]) * 1099511628211ull;
  for (size_t i = 0; i < inf.size(); ++i) h = (h ^ (unsigned)inf[i]) * 1099511628211ull;
  printf("    hash W+info %016llx\n", h);
}
template <class CF, int NG, int MINB, int RD, int RDB>
void run_ws(const Prob& P, Dev& d, const char* name, const std::vector<float2>& Wr, const std::vector<float>& gr, const std::vector<int>& ir) {
  size_t smem = NG * ws_shared_bytes<CF, RD, RDB>();
  auto k = chol_ws_kernel<CF, NG, MINB, RD, RDB>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k);
  int nb = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 64 * NG, smem);
  long long sg = (P.units + NG - 1) / NG;
  int grid = (int)(sg < 148LL * nb ? sg : 148LL * nb);
  CK(cudaMemset(d.W, 0xff, (size_t)P.units * P.S * P.N * 8));
  float us = timeit([&] { k<<<grid, 64 * NG, smem>>>(P.N, P.S, P.units, d.R, d.st, d.W, d.g, d.info); }, 10);
  CK(cudaGetLastError());
  report(P, name, us, fa.numRegs, fa.localSizeBytes, nb);
  std::vector<float2> W; std::vector<float> g; std::vector<int> inf;
  fetch(P, d, W, g, inf);
  long long dw = 0, dg = 0, di = 0;
  for (size_t i = 0; i < W.size(); ++i) dw += memcmp(&W[i], &Wr[i], 8) != 0;
  for (size_t i = 0; i < g.size(); ++i) dg += memcmp(&g[i], &gr[i], 4) != 0;
  for (size_t i = 0; i < inf.size(); ++i) di += inf[i] != ir[i];
  printf("    vs ref: W diff %lld  gamma diff %lld  info diff %lld  (info[7]=%d)\n", dw, dg, di, inf[7]);
}
template <class CF, int threads, int MINB>
void run_var(const Prob& P, Dev& d, const char* name, const std::vector<float2>& Wr, const std::vector<int>& ir) {
  size_t smem = (threads / CF::G) * chol_shared_bytes<CF>();
  auto k = chol_kernel<CF, threads, MINB>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k);
  int nb = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, threads, smem);
  long long per = threads / CF::G, sg = (P.units + per - 1) / per;
  int grid = (int)(sg < 148LL * nb ? sg : 148LL * nb);
  CK(cudaMemset(d.W, 0xff, (size_t)P.units * P.S * P.N * 8));
  float us = timeit([&] { k<<<grid, threads, smem>>>(P.N, P.S, P.units, d.R, d.st, d.W, d.g, d.info); }, 10);
  CK(cudaGetLastError());
  report(P, name, us, fa.numRegs, fa.localSizeBytes, nb);
  std::vector<float2> W; std::vector<float> g; std::vector<int> inf;
  fetch(P, d, W, g, inf);
  double maxe = 0; long long di = 0;
  for (long long u = 0; u < P.units; ++u) {
    di += inf[u] != ir[u];
    for (int kk = 0; kk < P.S; ++kk) {
      double num = 0, den = 0;
      for (int i = 0; i < P.N; ++i) {
        float2 a = W[(u * P.S + kk) * P.N + i], b = Wr[(u * P.S + kk) * P.N + i];
        num += (a.x - b.x) * (a.x - b.x) + (a.y - b.y) * (a.y - b.y); den += b.x * b.x + b.y * b.y;
      }
      double e = sqrt(num / (den + 1e-300)); if (!(e <= maxe)) maxe = e;
    }
  }
  printf("    vs ref: max rel %.2e  info diff %lld\n", maxe, di);
}
int main(int argc, char** argv) {
  const bool ref_only = argc > 1;
  for (int cfg = 0; cfg < 2; ++cfg) {
    const int N = cfg == 0 ? 56 : 30, S = 16, K = cfg == 0 ? 128 : 64;
    const long long units = cfg == 0 ? 65536 : 131072;
    Prob P = make(N, S, units, 512, K);
    Dev d;
    CK(cudaMalloc(&d.R, P.R.size() * 8)); CK(cudaMalloc(&d.st, P.st.size() * 8));
    CK(cudaMalloc(&d.W, (size_t)units * S * N * 8)); CK(cudaMalloc(&d.g, units * S * 4)); CK(cudaMalloc(&d.info, units * 4));
    CK(cudaMemcpy(d.R, P.R.data(), P.R.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d.st, P.st.data(), P.st.size() * 8, cudaMemcpyHostToDevice));
    std::vector<float2> W; std::vector<float> g; std::vector<int> inf;
    if (cfg == 0) {
      printf("== large N=56 S=16 units=%lld\n", units);
      using CF = CholCfg<4, 8, 14, 7, 2, false, 2>;
      run_ref<CF, 128, 2>(P, d, W, g, inf);
#ifdef VARS
      run_var<CholCfg<4, 8, 14, 7, 2, false, 2, true>, 128, 2>(P, d, "DBL 4x8 14x7 128x2", W, inf);
#endif
#ifndef NO_WS
      if (!ref_only) {
      run_ws<CF, 1, 6, 4, 4>(P, d, "ws ng1 mb6", W, g, inf);
      run_ws<CF, 1, 5, 4, 4>(P, d, "ws ng1 mb5", W, g, inf);
      run_ws<CF, 2, 3, 4, 4>(P, d, "ws ng2 mb3", W, g, inf);
      run_ws<CF, 1, 4, 4, 4>(P, d, "ws ng1 mb4", W, g, inf);
      }
#endif
    } else {
      printf("== medium N=30 S=16 units=%lld\n", units);
      using CF = CholCfg<4, 8, 8, 4, 2, false, 2>;
      run_ref<CF, 256, 2>(P, d, W, g, inf);
#ifdef VARS
      run_var<CholCfg<4, 8, 8, 4, 2, false, 2, true>, 256, 2>(P, d, "DBL 4x8 8x4 256x2", W, inf);
      run_var<CholCfg<4, 8, 8, 4, 2, false, 2, true>, 128, 3>(P, d, "DBL 4x8 8x4 128x3", W, inf);
#endif
#ifndef NO_WS
      if (!ref_only) {
      run_ws<CF, 1, 8, 4, 4>(P, d, "ws ng1 mb8", W, g, inf);
      run_ws<CF, 1, 6, 4, 4>(P, d, "ws ng1 mb6", W, g, inf);
      run_ws<CF, 2, 4, 4, 4>(P, d, "ws ng2 mb4", W, g, inf);
      }
#endif
    }
    cudaFree(d.R); cudaFree(d.st); cudaFree(d.W); cudaFree(d.g); cudaFree(d.info);
  }
  return 0;
}

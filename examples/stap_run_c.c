/* stap_run_c.c -- the whole STAP path from plain C through the C ABI (include/stap.h), no
 * Python: build a plan, copy a datacube and steering vectors to the device, run stap_run,
 * copy the beamformed outputs and the per-unit info back.
 *
 *   gcc -std=c11 -O2 -I include -I /usr/local/cuda/include examples/stap_run_c.c \
 *       -L paper_2203_06233_b200 -lstap -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,paper_2203_06233_b200 -o /tmp/stap_run_c
 *   /tmp/stap_run_c [out_prefix]
 *
 * Shape: BASELINE.json configs[1] (small: C=4, T=3, D=256, R=512, K=32, S=16), one cube, FP32.
 * The cube and the steering set come from a fixed xorshift generator; with an out_prefix the
 * program writes <prefix>_cube.bin, <prefix>_steer.bin, <prefix>_out.bin, <prefix>_info.bin
 * (raw little-endian complex64 / int32) so that a test can compare them with another path. */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "stap.h"

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      fprintf(stderr, "CUDA %s at line %d\n", cudaGetErrorString(e_), __LINE__); \
      return 1;                                                                \
    }                                                                          \
  } while (0)
#define SK(x)                                                                  \
  do {                                                                         \
    stap_status s_ = (x);                                                      \
    if (s_ != STAP_OK) {                                                       \
      fprintf(stderr, "%s at line %d\n", stap_status_string(s_), __LINE__);    \
      return 1;                                                                \
    }                                                                          \
  } while (0)

static unsigned long long rng = 0x9e3779b97f4a7c15ull;
static float urand(void) { /* xorshift64, uniform in [-1, 1) */
  rng ^= rng << 13;
  rng ^= rng >> 7;
  rng ^= rng << 17;
  return (float)((rng >> 40) * (1.0 / 8388608.0) - 1.0);
}

static int dump(const char* prefix, const char* name, const void* p, size_t bytes) {
  char path[512];
  snprintf(path, sizeof path, "%s_%s.bin", prefix, name);
  FILE* f = fopen(path, "wb");
  if (!f || fwrite(p, 1, bytes, f) != bytes) return 1;
  fclose(f);
  return 0;
}

int main(int argc, char** argv) {
  stap_params prm;
  memset(&prm, 0, sizeof prm);
  prm.n_chan = 4;
  prm.tdof = 3;
  prm.n_dop = 256;
  prm.n_range = 512;
  prm.training_block = 32;
  prm.n_steering = 16;
  prm.diag_load = 1e-2f;
  prm.dop_begin = 0;
  prm.dop_count = prm.n_dop;
  prm.cube_bin0 = 0;
  prm.cube_bins = prm.n_dop;
  prm.batch = 1;
  prm.device = 0;
  prm.path = STAP_PATH_AUTO;
  prm.precision = STAP_PREC_FP32;
  if (stap_abi_version() != STAP_ABI_VERSION) {
    fprintf(stderr, "header/library ABI mismatch\n");
    return 1;
  }
  stap_plan* plan = NULL;
  SK(stap_plan_create(&prm, &plan));
  printf("plan: %s\n", stap_plan_describe(plan));

  const int C = prm.n_chan, N = prm.n_chan * prm.tdof, D = prm.n_dop, R = prm.n_range, S = prm.n_steering;
  const int B = R / prm.training_block;
  const size_t n_cube = (size_t)D * C * R, n_steer = (size_t)S * N, n_out = (size_t)D * S * R, n_info = (size_t)D * B;
  stap_c64* h_cube = malloc(n_cube * sizeof(stap_c64));
  stap_c64* h_steer = malloc(n_steer * sizeof(stap_c64));
  stap_c64* h_out = malloc(n_out * sizeof(stap_c64));
  int32_t* h_info = malloc(n_info * sizeof(int32_t));
  if (!h_cube || !h_steer || !h_out || !h_info) return 1;
  for (size_t i = 0; i < n_cube; ++i) {
    h_cube[i].re = urand();
    h_cube[i].im = urand();
  }
  for (size_t i = 0; i < n_steer; ++i) {
    h_steer[i].re = urand();
    h_steer[i].im = urand();
  }

  CK(cudaSetDevice(prm.device));
  stap_c64 *d_cube, *d_steer, *d_out;
  int32_t* d_info;
  void* ws = NULL;
  size_t ws_bytes = 0;
  SK(stap_plan_workspace_bytes(plan, 0, &ws_bytes));
  CK(cudaMalloc((void**)&d_cube, n_cube * sizeof(stap_c64)));
  CK(cudaMalloc((void**)&d_steer, n_steer * sizeof(stap_c64)));
  CK(cudaMalloc((void**)&d_out, n_out * sizeof(stap_c64)));
  CK(cudaMalloc((void**)&d_info, n_info * sizeof(int32_t)));
  if (ws_bytes) CK(cudaMalloc(&ws, ws_bytes));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  CK(cudaMemcpyAsync(d_cube, h_cube, n_cube * sizeof(stap_c64), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_steer, h_steer, n_steer * sizeof(stap_c64), cudaMemcpyHostToDevice, st));
  SK(stap_run(plan, d_cube, d_steer, d_out, d_info, ws, ws_bytes, st));
  CK(cudaMemcpyAsync(h_out, d_out, n_out * sizeof(stap_c64), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h_info, d_info, n_info * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));

  double e = 0.0;
  long long bad = 0;
  for (size_t i = 0; i < n_out; ++i) e += (double)h_out[i].re * h_out[i].re + (double)h_out[i].im * h_out[i].im;
  for (size_t i = 0; i < n_info; ++i) bad += h_info[i] != 0;
  printf("out energy %.6e, units with info != 0: %lld of %zu\n", e, bad, n_info);

  if (argc > 1 && (dump(argv[1], "cube", h_cube, n_cube * sizeof(stap_c64)) ||
                   dump(argv[1], "steer", h_steer, n_steer * sizeof(stap_c64)) ||
                   dump(argv[1], "out", h_out, n_out * sizeof(stap_c64)) ||
                   dump(argv[1], "info", h_info, n_info * sizeof(int32_t)))) {
    fprintf(stderr, "cannot write %s_*.bin\n", argv[1]);
    return 1;
  }
  cudaStreamDestroy(st);
  cudaFree(d_cube);
  cudaFree(d_steer);
  cudaFree(d_out);
  cudaFree(d_info);
  if (ws) cudaFree(ws);
  SK(stap_plan_destroy(plan));
  free(h_cube);
  free(h_steer);
  free(h_out);
  free(h_info);
  return 0;
}

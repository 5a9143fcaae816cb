/* stap_comm_c.c -- the multi-GPU path from plain C through the C ABI (include/stap.h):
 * one process drives G = 2 GPUs (stap_comm_create); each GPU owns half of the Doppler bins of
 * one datacube (its cube buffer holds those bins plus the T-1 halo), runs stap_run on them, and
 * the library's in-place all-gather (stap_comm_allgather_out) leaves the whole Doppler-major
 * output on both GPUs.  The program checks, bitwise, that both gathered copies equal an
 * unsharded run of the whole cube on GPU 0, and exits 0 only then (2 when fewer than two GPUs).
 *
 *   gcc -std=c11 -O2 -I include -I /usr/local/cuda/include examples/stap_comm_c.c \
 *       -L paper_2203_06233_b200 -lstap -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,paper_2203_06233_b200 -o /tmp/stap_comm_c
 *
 * Shape: BASELINE.json configs[1] per GPU (small: C=4, T=3, R=512, K=32, S=16), global D = 512. */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "stap.h"

#define G 2
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

static unsigned long long rng = 0x2545f4914f6cdd1dull;
static float urand(void) {
  rng ^= rng << 13;
  rng ^= rng >> 7;
  rng ^= rng << 17;
  return (float)((rng >> 40) * (1.0 / 8388608.0) - 1.0);
}

static stap_params base_params(int D) {
  stap_params p;
  memset(&p, 0, sizeof p);
  p.n_chan = 4;
  p.tdof = 3;
  p.n_dop = D;
  p.n_range = 512;
  p.training_block = 32;
  p.n_steering = 16;
  p.diag_load = 1e-2f;
  p.dop_count = D;
  p.cube_bins = D;
  p.batch = 1;
  p.path = STAP_PATH_AUTO;
  p.precision = STAP_PREC_FP32;
  return p;
}

int main(void) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < G) {
    printf("needs %d GPUs\n", G);
    return 2;
  }
  const int D = 512, Dl = D / G, C = 4, T = 3, h = (T - 1) / 2, R = 512, S = 16, N = C * T;
  const size_t row = (size_t)C * R;                  /* complex64 per Doppler bin of the cube */
  const size_t slice = (size_t)Dl * S * R;           /* complex64 per rank of the output */
  stap_c64* h_cube = malloc((size_t)D * row * sizeof(stap_c64));
  stap_c64* h_steer = malloc((size_t)S * N * sizeof(stap_c64));
  stap_c64* h_ref = malloc((size_t)D * S * R * sizeof(stap_c64));
  stap_c64* h_got = malloc((size_t)G * slice * sizeof(stap_c64));
  if (!h_cube || !h_steer || !h_ref || !h_got) return 1;
  for (size_t i = 0; i < (size_t)D * row; ++i) {
    h_cube[i].re = urand();
    h_cube[i].im = urand();
  }
  for (int i = 0; i < S * N; ++i) {
    h_steer[i].re = urand();
    h_steer[i].im = urand();
  }

  /* reference: the whole cube on GPU 0 */
  {
    stap_params p = base_params(D);
    stap_plan* plan;
    SK(stap_plan_create(&p, &plan));
    CK(cudaSetDevice(0));
    stap_c64 *d_cube, *d_steer, *d_out;
    int32_t* d_info;
    void* ws = NULL;
    size_t wsb = 0;
    SK(stap_plan_workspace_bytes(plan, 0, &wsb));
    CK(cudaMalloc((void**)&d_cube, (size_t)D * row * sizeof(stap_c64)));
    CK(cudaMalloc((void**)&d_steer, (size_t)S * N * sizeof(stap_c64)));
    CK(cudaMalloc((void**)&d_out, (size_t)D * S * R * sizeof(stap_c64)));
    CK(cudaMalloc((void**)&d_info, (size_t)D * (R / 32) * sizeof(int32_t)));
    if (wsb) CK(cudaMalloc(&ws, wsb));
    CK(cudaMemcpy(d_cube, h_cube, (size_t)D * row * sizeof(stap_c64), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_steer, h_steer, (size_t)S * N * sizeof(stap_c64), cudaMemcpyHostToDevice));
    SK(stap_run(plan, d_cube, d_steer, d_out, d_info, ws, wsb, 0));
    CK(cudaMemcpy(h_ref, d_out, (size_t)D * S * R * sizeof(stap_c64), cudaMemcpyDeviceToHost));
    cudaFree(d_cube);
    cudaFree(d_steer);
    cudaFree(d_out);
    cudaFree(d_info);
    if (ws) cudaFree(ws);
    SK(stap_plan_destroy(plan));
  }

  /* sharded: rank r owns bins [r Dl, (r+1) Dl); its cube buffer starts at bin r Dl - h (mod D) */
  const int32_t devices[G] = {0, 1};
  stap_comm* comm;
  SK(stap_comm_create(G, devices, &comm));
  stap_plan* plans[G];
  stap_c64* outs[G];
  cudaStream_t streams[G];
  stap_c64 *d_cube[G], *d_steer[G];
  int32_t* d_info[G];
  void* ws[G];
  for (int r = 0; r < G; ++r) {
    stap_params p = base_params(D);
    p.dop_begin = r * Dl;
    p.dop_count = Dl;
    p.cube_bin0 = ((r * Dl - h) % D + D) % D;
    p.cube_bins = Dl + T - 1;
    p.device = devices[r];
    SK(stap_plan_create(&p, &plans[r]));
    CK(cudaSetDevice(devices[r]));
    CK(cudaStreamCreate(&streams[r]));
    size_t wsb = 0;
    SK(stap_plan_workspace_bytes(plans[r], 0, &wsb));
    ws[r] = NULL;
    if (wsb) CK(cudaMalloc(&ws[r], wsb));
    CK(cudaMalloc((void**)&d_cube[r], (size_t)p.cube_bins * row * sizeof(stap_c64)));
    CK(cudaMalloc((void**)&d_steer[r], (size_t)S * N * sizeof(stap_c64)));
    CK(cudaMalloc((void**)&outs[r], (size_t)G * slice * sizeof(stap_c64)));
    CK(cudaMalloc((void**)&d_info[r], (size_t)Dl * (R / 32) * sizeof(int32_t)));
    for (int w = 0; w < p.cube_bins; ++w) { /* the window rows, wrapping mod D */
      const int bin = (p.cube_bin0 + w) % D;
      CK(cudaMemcpy(d_cube[r] + (size_t)w * row, h_cube + (size_t)bin * row, row * sizeof(stap_c64),
                    cudaMemcpyHostToDevice));
    }
    CK(cudaMemcpy(d_steer[r], h_steer, (size_t)S * N * sizeof(stap_c64), cudaMemcpyHostToDevice));
    SK(stap_run(plans[r], d_cube[r], d_steer[r], outs[r] + (size_t)r * slice, d_info[r], ws[r], wsb, streams[r]));
  }
  SK(stap_comm_allgather_out(comm, outs, (const stap_plan* const*)plans, streams));

  int ok = 1;
  for (int r = 0; r < G; ++r) {
    CK(cudaSetDevice(devices[r]));
    CK(cudaStreamSynchronize(streams[r]));
    CK(cudaMemcpy(h_got, outs[r], (size_t)G * slice * sizeof(stap_c64), cudaMemcpyDeviceToHost));
    const int same = memcmp(h_got, h_ref, (size_t)G * slice * sizeof(stap_c64)) == 0;
    printf("GPU %d: gathered output %s the unsharded run\n", devices[r], same ? "bitwise equals" : "DIFFERS from");
    ok &= same;
  }
  for (int r = 0; r < G; ++r) {
    cudaSetDevice(devices[r]);
    cudaStreamDestroy(streams[r]);
    cudaFree(d_cube[r]);
    cudaFree(d_steer[r]);
    cudaFree(outs[r]);
    cudaFree(d_info[r]);
    if (ws[r]) cudaFree(ws[r]);
    stap_plan_destroy(plans[r]);
  }
  SK(stap_comm_destroy(comm));
  free(h_cube);
  free(h_steer);
  free(h_ref);
  free(h_got);
  return ok ? 0 : 1;
}

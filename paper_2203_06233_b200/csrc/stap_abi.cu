// stap_abi.cu -- host side of libstap.so: plan validation, launch-shape
// selection and the extern "C" entry points declared in include/stap.h.
//
// Nothing here does arithmetic of the method; every step runs in the kernels
// of cov.cuh / cov_tc.cuh (K1), chol.cuh / solve_small.cuh (K2), apply.cuh / apply_tc.cuh
// (K3) and fused.cuh (K4).  There
// is no CPU path: without an sm_100 device every call returns an error.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>

#include <cudaTypedefs.h>

#include "../../include/stap.h"
#include "internal.h"
#include "apply.cuh"
#include "apply_tc.cuh"
#include "cov.cuh"
#include "cov_tc.cuh"
#include "doppler.cuh"
#include "fused.cuh"
#include "chol.cuh"
#include "solve_small.cuh"

using namespace stapk;

struct stap_plan {
  stap_params prm;
  KParams kp;
  long long units;  // batch * dop_count * B
  // K1
  int cov_P, cov_threads, cov_runs;
  size_t cov_smem;
  int cov_tc, cov_tc_grid, cov_tc_tiles;  // tcgen05 3xTF32 covariance (cov_tc.cuh) when supported
  CovTcGeom cov_tc_geom;
  size_t cov_tc_smem;
  // K2
  CholSel solve_sel;             // N >= 13: chol.cuh
  int solve_small, solve_lanes;  // no chol_select instantiation: solve_small.cuh with `solve_lanes` lanes per matrix
  int solve_grid;
  size_t solve_smem;
  // K3
  int apply_tpu, apply_upc, apply_smax, apply_grid;
  int apply_tc, apply_tc_grid, apply_tc_ns;  // tcgen05 3xTF32 apply (apply_tc.cuh) when supported
  size_t apply_tc_smem;
  size_t apply_smem;
  // K4 (fused) selection
  int fused;  // 1 if stap_run uses the fused kernel
  FusedCfg fcfg;
  // staged workspace layout
  size_t ws_cov, ws_w, ws_g, ws_total;
  size_t cube_bytes, steer_bytes, out_bytes, info_bytes;
  char desc[160];
  // stap_run_host pipelining: the batch in io_nch chunks run by a child plan (batch / io_nch),
  // host->device copies, kernels and device->host copies of different chunks overlapped
  stap_plan* io_child = nullptr;
  int io_nch = 0;
  cudaStream_t io_s[2] = {nullptr, nullptr};
  cudaEvent_t io_ev[2 + 2 * 8] = {};
};

namespace {
void plan_free(stap_plan* pl) {
  if (!pl) return;
  if (pl->io_nch) {
    for (cudaEvent_t& e : pl->io_ev)
      if (e) cudaEventDestroy(e);
    for (cudaStream_t& q : pl->io_s)
      if (q) cudaStreamDestroy(q);
  }
  plan_free(pl->io_child);
  delete pl;
}
}  // namespace

namespace {

const size_t kSmemCap = 227 * 1024;
// a 16-byte aligned stand-in address for the plan-time tensor-map trial encode (never dereferenced)
const float2* const kTrialCube = reinterpret_cast<const float2*>(uintptr_t{1} << 20);

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) return;
    if (prev != dev && cudaSetDevice(dev) != cudaSuccess) return;
    ok = true;
  }
  ~DeviceGuard() {
    if (ok && prev >= 0) {
      int cur = -1;
      if (cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
  }
};

template <int C>
void cov_attr(size_t smem) {
  cudaFuncSetAttribute(cov_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t set_cov_attr(int C, size_t smem) {
  switch (C) {
    case 1: cov_attr<1>(smem); break;
    case 2: cov_attr<2>(smem); break;
    case 3: cov_attr<3>(smem); break;
    case 4: cov_attr<4>(smem); break;
    case 5: cov_attr<5>(smem); break;
    case 6: cov_attr<6>(smem); break;
    case 7: cov_attr<7>(smem); break;
    case 8: cov_attr<8>(smem); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// cuTensorMapEncodeTiled from the driver, without linking libcuda
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// the cube as a 2-D fp32 tensor [batch*nbins*C rows][2R floats] with box {bx floats, by rows}
bool encode_cube_map(const KParams& k, const float2* cube, CUtensorMap* map, int bx, int by,
                     CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_NONE) {
  const PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)2 * k.R, (cuuint64_t)k.batch * k.nbins * k.C};
  const cuuint64_t strides[1] = {(cuuint64_t)k.R * 8};
  const cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)by}, estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float2*>(cube), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// the two tensor maps the tcgen05 stages build per call (any 16-byte aligned cube)
bool encode_cov_tc_map(const stap_plan* pl, const float2* cube, CUtensorMap* m) {
  return encode_cube_map(pl->kp, cube, m, 32, pl->cov_tc_geom.MB * pl->kp.C, CU_TENSOR_MAP_SWIZZLE_128B);
}
bool encode_apply_tc_map(const stap_plan* pl, const float2* cube, CUtensorMap* m) {
  return encode_cube_map(pl->kp, cube, m, 128, pl->kp.C);
}

template <int C>
void cov_launch_t(const stap_plan* pl, const float2* cube, float2* cov, cudaStream_t st) {
  dim3 grid(pl->cov_runs, pl->kp.B, pl->kp.batch);
  cov_kernel<C><<<grid, pl->cov_threads, pl->cov_smem, st>>>(pl->kp, cube, cov, pl->cov_P);
}

// K1 on the kernel the plan chose (tcgen05 3xTF32 only under STAP_PREC_TF32X3); a tensor map
// that cannot be encoded is an error, never a silent switch of arithmetic.
stap_status cov_launch(const stap_plan* pl, const float2* cube, float2* cov, cudaStream_t st) {
  if (pl->cov_tc) {
    CUtensorMap msw;
    if (!encode_cov_tc_map(pl, cube, &msw)) return STAP_ERR_CUDA;
    cov_tc_kernel<<<pl->cov_tc_grid, kCovTcThreads, pl->cov_tc_smem, st>>>(msw, pl->kp, cube, cov, pl->cov_tc_tiles,
                                                                           pl->cov_tc_geom);
    return STAP_OK;
  }
  switch (pl->kp.C) {
    case 1: cov_launch_t<1>(pl, cube, cov, st); break;
    case 2: cov_launch_t<2>(pl, cube, cov, st); break;
    case 3: cov_launch_t<3>(pl, cube, cov, st); break;
    case 4: cov_launch_t<4>(pl, cube, cov, st); break;
    case 5: cov_launch_t<5>(pl, cube, cov, st); break;
    case 6: cov_launch_t<6>(pl, cube, cov, st); break;
    case 7: cov_launch_t<7>(pl, cube, cov, st); break;
    case 8: cov_launch_t<8>(pl, cube, cov, st); break;
  }
  return STAP_OK;
}

// K3 instantiations: SIMT by SMAX, tcgen05 by KS = ceil(N/8); each plain or REMOTE (multicast /
// peer-copy stores), the plain ones compiled with ordinary stores only
template <int SMAX, bool RM>
void apply_launch_t(const stap_plan* pl, const float2* cube, const float2* w, float2* out, cudaStream_t st) {
  apply_kernel<SMAX, RM><<<pl->apply_grid, pl->apply_upc * pl->apply_tpu, pl->apply_smem, st>>>(
      pl->kp, cube, w, out, pl->apply_tpu, pl->apply_upc, pl->units);
}
template <int KS, bool RM>
void apply_tc_launch_t(const stap_plan* pl, const CUtensorMap& map, const float2* w, float2* out, cudaStream_t st) {
  apply_tc_kernel<KS, RM><<<pl->apply_tc_grid, kApplyTcThreads, pl->apply_tc_smem, st>>>(map, pl->kp, w, out,
                                                                                          (int)pl->units, pl->apply_tc_ns);
}
template <bool RM>
void apply_tc_dispatch(const stap_plan* pl, const CUtensorMap& map, const float2* w, float2* out, cudaStream_t st) {
  switch ((pl->kp.N + 7) / 8) {
    case 1: apply_tc_launch_t<1, RM>(pl, map, w, out, st); break;
    case 2: apply_tc_launch_t<2, RM>(pl, map, w, out, st); break;
    case 3: apply_tc_launch_t<3, RM>(pl, map, w, out, st); break;
    case 4: apply_tc_launch_t<4, RM>(pl, map, w, out, st); break;
    case 5: apply_tc_launch_t<5, RM>(pl, map, w, out, st); break;
    case 6: apply_tc_launch_t<6, RM>(pl, map, w, out, st); break;
    case 7: apply_tc_launch_t<7, RM>(pl, map, w, out, st); break;
    case 8: apply_tc_launch_t<8, RM>(pl, map, w, out, st); break;
  }
}
template <bool RM>
void apply_simt_dispatch(const stap_plan* pl, const float2* cube, const float2* w, float2* out, cudaStream_t st) {
  switch (pl->apply_smax) {
    case 2: apply_launch_t<2, RM>(pl, cube, w, out, st); break;
    case 4: apply_launch_t<4, RM>(pl, cube, w, out, st); break;
    case 8: apply_launch_t<8, RM>(pl, cube, w, out, st); break;
    case 16: apply_launch_t<16, RM>(pl, cube, w, out, st); break;
    case 32: apply_launch_t<32, RM>(pl, cube, w, out, st); break;
  }
}
template <int KS>
void apply_tc_attr_t(size_t smem) {
  cudaFuncSetAttribute(apply_tc_kernel<KS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(apply_tc_kernel<KS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}
void apply_tc_attr(int N, size_t smem) {
  switch ((N + 7) / 8) {
    case 1: apply_tc_attr_t<1>(smem); break;
    case 2: apply_tc_attr_t<2>(smem); break;
    case 3: apply_tc_attr_t<3>(smem); break;
    case 4: apply_tc_attr_t<4>(smem); break;
    case 5: apply_tc_attr_t<5>(smem); break;
    case 6: apply_tc_attr_t<6>(smem); break;
    case 7: apply_tc_attr_t<7>(smem); break;
    case 8: apply_tc_attr_t<8>(smem); break;
  }
}

stap_status apply_launch(const stap_plan* pl, const float2* cube, const float2* w, float2* out, cudaStream_t st) {
  const bool rm = pl->kp.y_mc || pl->kp.y_np;
  if (pl->apply_tc) {
    CUtensorMap map;
    if (!encode_apply_tc_map(pl, cube, &map)) return STAP_ERR_CUDA;
    if (rm)
      apply_tc_dispatch<true>(pl, map, w, out, st);
    else
      apply_tc_dispatch<false>(pl, map, w, out, st);
    return STAP_OK;
  }
  if (rm)
    apply_simt_dispatch<true>(pl, cube, w, out, st);
  else
    apply_simt_dispatch<false>(pl, cube, w, out, st);
  return STAP_OK;
}

template <int SMAX>
void apply_attr(size_t smem) {
  cudaFuncSetAttribute(apply_kernel<SMAX, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(apply_kernel<SMAX, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

void set_apply_attr(int smax, size_t smem) {
  switch (smax) {
    case 2: apply_attr<2>(smem); break;
    case 4: apply_attr<4>(smem); break;
    case 8: apply_attr<8>(smem); break;
    case 16: apply_attr<16>(smem); break;
    case 32: apply_attr<32>(smem); break;
  }
}

void solve_dispatch(const stap_plan* pl, const float2* cov, const float2* steer, float2* w, float* g, int32_t* info,
                    cudaStream_t st) {
  if (pl->solve_small)
    solve_small_launch(pl->kp.N, pl->solve_lanes, pl->solve_grid, 256, pl->solve_smem, st, pl->kp.S, pl->units, cov,
                       steer, w, g, info);
  else
    solve_chol_launch(pl->solve_sel, pl->solve_grid, st, pl->kp.N, pl->kp.S, pl->units, cov, steer, w, g, info);
}

stap_status check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "libstap: launch failed: %s\n", cudaGetErrorString(e));
    return STAP_ERR_CUDA;
  }
  return STAP_OK;
}

stap_status staged_run(const stap_plan* pl, const float2* cube, const float2* steer, float2* out,
                       int32_t* info, void* ws, cudaStream_t st) {
  char* w = static_cast<char*>(ws);
  float2* cov = reinterpret_cast<float2*>(w);
  float2* wts = reinterpret_cast<float2*>(w + pl->ws_cov);
  float* gam = reinterpret_cast<float*>(w + pl->ws_cov + pl->ws_w);
  stap_status s = cov_launch(pl, cube, cov, st);
  if (s != STAP_OK) return s;
  solve_dispatch(pl, cov, steer, wts, gam, info, st);
  s = apply_launch(pl, cube, wts, out, st);
  if (s != STAP_OK) return s;
  return check_launch();
}

}  // namespace

namespace stapk {
bool plan_out_geom(const stap_plan* pl, PlanOutGeom* g) {
  if (!pl || !g) return false;
  g->batch = pl->prm.batch;
  g->dop_count = pl->prm.dop_count;
  g->S = pl->prm.n_steering;
  g->R = pl->prm.n_range;
  g->device = pl->prm.device;
  g->out_bytes = pl->out_bytes;
  return true;
}
}  // namespace stapk

extern "C" {

int32_t stap_abi_version(void) { return STAP_ABI_VERSION; }

#ifdef COVTC_PROF
extern "C" int stap_debug_covtc_prof(unsigned long long* out) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(out, stapk::g_covtc_prof, sizeof(unsigned long long) * 8);
}
#endif

const char* stap_status_string(stap_status s) {
  switch (s) {
    case STAP_OK: return "STAP_OK";
    case STAP_ERR_NULL_ARG: return "STAP_ERR_NULL_ARG: a required pointer is NULL";
    case STAP_ERR_BAD_DIMS: return "STAP_ERR_BAD_DIMS: invalid dimensions, shard, cube window or workspace";
    case STAP_ERR_UNSUPPORTED: return "STAP_ERR_UNSUPPORTED: valid but not implemented (N>64, S>32, C>8, odd K, window > smem)";
    case STAP_ERR_MISALIGNED: return "STAP_ERR_MISALIGNED: device pointer not 16-byte aligned";
    case STAP_ERR_CUDA: return "STAP_ERR_CUDA: CUDA runtime or launch error";
    case STAP_ERR_NCCL: return "STAP_ERR_NCCL: NCCL unavailable, or an NCCL / IPC call failed";
    case STAP_ERR_DEVICE: return "STAP_ERR_DEVICE: no sm_100 device at the plan's ordinal";
  }
  return "STAP_ERR_UNKNOWN";
}

static stap_status plan_create_impl(const stap_params* p, stap_plan** out_plan, bool with_io);

stap_status stap_plan_create(const stap_params* p, stap_plan** out_plan) { return plan_create_impl(p, out_plan, true); }

static stap_status plan_create_impl(const stap_params* p, stap_plan** out_plan, bool with_io) {
  if (!p || !out_plan) return STAP_ERR_NULL_ARG;
  *out_plan = nullptr;
  const int C = p->n_chan, T = p->tdof, D = p->n_dop, R = p->n_range, K = p->training_block,
            S = p->n_steering;
  if (C <= 0 || T <= 0 || D <= 0 || R <= 0 || K <= 0 || S <= 0 || p->batch <= 0) return STAP_ERR_BAD_DIMS;
  if (p->path < STAP_PATH_AUTO || p->path > STAP_PATH_STAGED) return STAP_ERR_BAD_DIMS;
  if (p->precision != STAP_PREC_FP32 && p->precision != STAP_PREC_TF32X3) return STAP_ERR_BAD_DIMS;
  if (p->out_multicast != 0 && p->out_multicast != 1) return STAP_ERR_BAD_DIMS;
  if (p->out_n_peers < 0 || p->out_n_peers > 7 || (p->out_n_peers > 0 && p->out_multicast)) return STAP_ERR_BAD_DIMS;
  for (int i = 0; i < p->out_n_peers; ++i)
    if (p->out_peer_offset[i] % 16 != 0) return STAP_ERR_MISALIGNED;
  if (R % K != 0 || T > D) return STAP_ERR_BAD_DIMS;
  if (!(p->diag_load >= 0.0f) || !std::isfinite(p->diag_load)) return STAP_ERR_BAD_DIMS;
  if (p->dop_begin < 0 || p->dop_count <= 0 || (long long)p->dop_begin + p->dop_count > D)
    return STAP_ERR_BAD_DIMS;
  if (p->cube_bins <= 0 || p->cube_bins > D || p->cube_bin0 < 0 || p->cube_bin0 >= D) return STAP_ERR_BAD_DIMS;
  const int h = (T - 1) / 2;
  if (p->cube_bins < D) {
    long long off = ((long long)p->dop_begin - h - p->cube_bin0) % D;
    if (off < 0) off += D;
    if (off + p->dop_count + T - 1 > p->cube_bins) return STAP_ERR_BAD_DIMS;
  }
  const int N = C * T;
  if (N > 64 || S > 32 || C > 8 || (K & 1) || K > 1024) return STAP_ERR_UNSUPPORTED;

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || p->device < 0 || p->device >= ndev) {
    cudaGetLastError();
    return STAP_ERR_DEVICE;
  }
  int major = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, p->device) != cudaSuccess || major != 10)
    return STAP_ERR_DEVICE;
  {
    // the tensor-map encoder (a driver call, used below to decide the tcgen05 stages) needs the
    // device's primary context: create it here, so that a plan made before any other CUDA call
    // in the process selects exactly the kernels any later plan of the same parameters does
    DeviceGuard g(p->device);
    if (!g.ok || cudaFree(nullptr) != cudaSuccess) {
      cudaGetLastError();
      return STAP_ERR_DEVICE;
    }
  }

  stap_plan* pl = new (std::nothrow) stap_plan();
  if (!pl) return STAP_ERR_CUDA;
  pl->prm = *p;
  KParams& kp = pl->kp;
  kp.C = C; kp.T = T; kp.N = N; kp.D = D; kp.R = R; kp.K = K; kp.B = R / K; kp.S = S; kp.h = h;
  kp.lam = p->diag_load;
  kp.dop_begin = p->dop_begin; kp.dop_count = p->dop_count;
  kp.bin0 = p->cube_bin0; kp.nbins = p->cube_bins; kp.batch = p->batch;
  kp.cube_stride = (long long)p->cube_bins * C * R;
  kp.y_mc = p->out_multicast;
  kp.y_np = p->out_n_peers;
  for (int i = 0; i < 7; ++i) kp.y_off[i] = i < p->out_n_peers ? (long long)p->out_peer_offset[i] : 0;
  pl->units = (long long)p->batch * p->dop_count * kp.B;

  // K1: bins per CTA -- the largest run whose lag blocks fit 256 threads with
  // <= 113 KB of shared memory (two CTAs per SM), else the largest that fits at all.
  int P = 0;
  for (int q = 1; q <= p->dop_count && q <= 128; ++q) {
    int thr = (cov_tpb(C) * cov_blocks(T, q + T - 1) + 31) / 32 * 32;
    if (thr > 256 || cov_smem_bytes(C, T, K, q) > 113 * 1024) break;
    P = q;
  }
  if (P == 0) {
    int thr = (cov_tpb(C) * cov_blocks(T, T) + 31) / 32 * 32;
    if (thr > 256 || cov_smem_bytes(C, T, K, 1) > kSmemCap) {
      delete pl;
      return STAP_ERR_UNSUPPORTED;
    }
    P = 1;
  }
  pl->cov_P = P;
  pl->cov_threads = (cov_tpb(C) * cov_blocks(T, P + T - 1) + 31) / 32 * 32;
  pl->cov_runs = (p->dop_count + P - 1) / P;
  pl->cov_smem = cov_smem_bytes(C, T, K, P);
  {
    // tcgen05 3xTF32 covariance only when the caller asked for it (stap_params.precision) and the
    // shape and a trial tensor-map encode allow it; decided here, once, for every call of the plan
    pl->cov_tc_geom = cov_tc_geom(C, T, N, p->dop_count);
    pl->cov_tc_tiles = p->batch * kp.B * pl->cov_tc_geom.ntd;
    // the deepest TMA ring (2..4 chunks) that fits (measured: 3 stages large 565 -> 560 us,
    // 4 stages medium 442 -> 434 us)
    for (int ns = 4; ns >= 2; --ns) {
      pl->cov_tc_geom.NS = ns;
      pl->cov_tc_smem = cov_tc_smem(N, pl->cov_tc_geom.RS, pl->cov_tc_geom.OB, ns).total;
      if (pl->cov_tc_smem <= kSmemCap) break;
    }
    pl->cov_tc = (p->precision == STAP_PREC_TF32X3 && cov_tc_supported(C, T, N, K) && tensor_map_encoder() &&
                  pl->cov_tc_smem <= kSmemCap)
                     ? 1
                     : 0;
    CUtensorMap trial;
    if (pl->cov_tc && !encode_cov_tc_map(pl, kTrialCube, &trial)) pl->cov_tc = 0;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, p->device);
    pl->cov_tc_grid = pl->cov_tc_tiles < nsm ? pl->cov_tc_tiles : nsm;  // persistent, one CTA per SM
  }

  // K2: chol.cuh's lane-group layout where chol_select has an instantiation for (N, S)
  // (N >= 13); below that solve_small (two matrices per warp for S <= 16).
  // Persistent grids: the blocks resident on every SM.
  const bool chol_ok = chol_select(N, S, &pl->solve_sel);
  if (!chol_ok && N > 16) {
    delete pl;
    return STAP_ERR_UNSUPPORTED;
  }
  pl->solve_small = chol_ok ? 0 : 1;
  {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, p->device);
    if (pl->solve_small) {
      pl->solve_lanes = S <= 16 ? 16 : 32;
      const int per_cta = 8 * (32 / pl->solve_lanes);  // matrices per 256-thread CTA
      pl->solve_smem = solve_small_smem(N, pl->solve_lanes, 256);
      long long sg = (pl->units + per_cta - 1) / per_cta;
      pl->solve_grid = (int)(sg < 148LL * 64 ? sg : 148LL * 64);
    } else {
      pl->solve_smem = pl->solve_sel.smem;
      const long long sg = (pl->units + pl->solve_sel.groups - 1) / pl->solve_sel.groups;
      const long long cap = (long long)nsm * pl->solve_sel.min_blocks;
      pl->solve_grid = (int)(sg < cap ? sg : cap);
    }
    if (pl->solve_smem > kSmemCap) {
      delete pl;
      return STAP_ERR_UNSUPPORTED;
    }
  }

  // K3
  pl->apply_tpu = apply_tpu(K);
  pl->apply_upc = 128 / pl->apply_tpu;
  pl->apply_smax = S <= 2 ? 2 : S <= 4 ? 4 : S <= 8 ? 8 : S <= 16 ? 16 : 32;
  pl->apply_smem = apply_smem_bytes(N, pl->apply_smax, pl->apply_upc);
  pl->apply_grid = (int)((pl->units + pl->apply_upc - 1) / pl->apply_upc);
  {
    pl->apply_tc = (p->precision == STAP_PREC_TF32X3 && apply_tc_supported(N, S, K) && pl->units < (1LL << 30) &&
                    tensor_map_encoder())
                       ? 1
                       : 0;
    CUtensorMap trial;
    if (pl->apply_tc && !encode_apply_tc_map(pl, kTrialCube, &trial)) pl->apply_tc = 0;
    pl->apply_tc_ns = apply_tc_stages(N);
    pl->apply_tc_smem = apply_tc_smem_bytes(N);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, p->device);
    const long long g = 2LL * nsm;  // persistent: two CTAs per SM, each walking whole units
    pl->apply_tc_grid = (int)(pl->units < g ? pl->units : g);
  }

  // K4: fused single-kernel path when it fits and the caller's path allows it.  AUTO
  // prefers the staged path when both tensor-core stages apply (K1 and K3 on tcgen05;
  // medium, 16 cubes on B200: staged 2.30 ms vs fused 2.48 ms per step), else the fused
  // kernel when it fits (small); shapes it cannot hold (large) run staged.
  const bool fits = fused_configure(kp, &pl->fcfg);
  if (p->path == STAP_PATH_FUSED && !fits) {
    delete pl;
    return STAP_ERR_UNSUPPORTED;
  }
  const bool tc_staged = pl->cov_tc && pl->apply_tc;
  pl->fused = (fits && (p->path == STAP_PATH_FUSED || (p->path == STAP_PATH_AUTO && !tc_staged))) ? 1 : 0;

  // staged workspace
  const long long NN = (long long)N * N;
  pl->ws_cov = align_up((size_t)pl->units * NN * 8, 256);
  pl->ws_w = align_up((size_t)pl->units * S * N * 8, 256);
  pl->ws_g = align_up((size_t)pl->units * S * 4, 256);
  pl->ws_total = pl->fused ? 0 : pl->ws_cov + pl->ws_w + pl->ws_g;
  pl->cube_bytes = (size_t)p->batch * kp.cube_stride * 8;
  pl->steer_bytes = (size_t)S * N * 8;
  pl->out_bytes = (size_t)p->batch * p->dop_count * S * (size_t)R * 8;
  pl->info_bytes = (size_t)pl->units * 4;

  {
    DeviceGuard g(p->device);
    if (!g.ok) {
      delete pl;
      return STAP_ERR_DEVICE;
    }
    if (set_cov_attr(C, pl->cov_smem) != cudaSuccess ||
        (pl->cov_tc && cudaFuncSetAttribute(cov_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)pl->cov_tc_smem) != cudaSuccess)) {
      delete pl;
      cudaGetLastError();
      return STAP_ERR_CUDA;
    }
    if (pl->solve_small)
      solve_small_set_attr(N, pl->solve_lanes, pl->solve_smem);
    else
      solve_chol_set_attr(pl->solve_sel);
    set_apply_attr(pl->apply_smax, pl->apply_smem);
    if (pl->apply_tc)
      apply_tc_attr(N, pl->apply_tc_smem);
    if (pl->fused) fused_set_attr(pl->fcfg);
    if (cudaGetLastError() != cudaSuccess) {
      delete pl;
      return STAP_ERR_CUDA;
    }
  }
  if (pl->fused)
    snprintf(pl->desc, sizeof pl->desc, "fused:%s", pl->fcfg.name);
  else
    snprintf(pl->desc, sizeof pl->desc, "staged:cov(%s,P=%d,thr=%d,smem=%zu)+solve(id=%d,G=%d)+apply(%s,tpu=%d,upc=%d)",
             pl->cov_tc ? "tcgen05-3xtf32" : "simt", pl->cov_P, pl->cov_threads, pl->cov_smem, pl->solve_small ? 100 + N : pl->solve_sel.id,
             pl->solve_small ? pl->solve_lanes : pl->solve_sel.threads / pl->solve_sel.groups, pl->apply_tc ? "tcgen05-3xtf32" : "simt", pl->apply_tpu,
             pl->apply_upc);
  // host-I/O pipelining (stap_run_host): up to 8 equal chunks of whole cubes.  A chunk count
  // whose per-chunk buffers would not keep 16-byte offsets is skipped (e.g. an odd number of
  // info words per chunk); with none left, stap_run_host runs unchunked.
  const int M = p->batch;
  for (int nch = 8; with_io && nch > 1 && !pl->io_nch; nch >>= 1) {
    if (M % nch) continue;
    stap_params cp = *p;
    cp.batch = M / nch;
    stap_plan* child = nullptr;
    const bool fit = plan_create_impl(&cp, &child, false) == STAP_OK && child->info_bytes % 16 == 0 &&
                     child->cube_bytes % 16 == 0 && child->out_bytes % 16 == 0;
    if (!fit) {
      plan_free(child);
      continue;
    }
    DeviceGuard g(p->device);
    pl->io_child = child;
    pl->io_nch = nch;
    bool ok = g.ok;
    for (cudaStream_t& q : pl->io_s) ok = ok && cudaStreamCreateWithFlags(&q, cudaStreamNonBlocking) == cudaSuccess;
    for (cudaEvent_t& e : pl->io_ev) ok = ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
      plan_free(pl);
      cudaGetLastError();
      return STAP_ERR_CUDA;
    }
  }
  *out_plan = pl;
  return STAP_OK;
}

stap_status stap_plan_destroy(stap_plan* plan) {
  plan_free(plan);
  return STAP_OK;
}

stap_status stap_plan_workspace_bytes(const stap_plan* pl, int32_t host_io, size_t* bytes) {
  if (!pl || !bytes) return STAP_ERR_NULL_ARG;
  size_t b = pl->ws_total;
  if (host_io)
    b += align_up(pl->cube_bytes, 256) + align_up(pl->steer_bytes, 256) + align_up(pl->out_bytes, 256) +
         align_up(pl->info_bytes, 256);
  *bytes = b;
  return STAP_OK;
}

const char* stap_plan_describe(const stap_plan* pl) { return pl ? pl->desc : "(null plan)"; }

stap_status stap_doppler(const stap_plan* pl, const float* window, const stap_c64* raw, stap_c64* cube,
                         cudaStream_t st) {
  if (!pl || !window || !raw || !cube) return STAP_ERR_NULL_ARG;
  const stap_params& p = pl->prm;
  const int D = p.n_dop;
  if (p.dop_begin != 0 || p.dop_count != D || p.cube_bins != D || p.cube_bin0 != 0 || D < 2 || D > 8192 ||
      (D & (D - 1)))
    return STAP_ERR_UNSUPPORTED;
  if (!aligned16(raw) || !aligned16(cube) || (reinterpret_cast<uintptr_t>(window) & 3u)) return STAP_ERR_MISALIGNED;
  DeviceGuard g(p.device);
  if (!g.ok) return STAP_ERR_DEVICE;
  if (D >= 16 && D <= 1024) {  // K0b, the two-level register FFT
    int logD = 0;
    while ((1 << logD) < D) ++logD;
    const int L1 = 1 << ((logD + 1) / 2), L2 = D / L1;
    int rc = 16;
    while (rc > 4 && (doppler2_smem(L1, L2, rc) > kDoppler2MaxSmem || p.n_range % rc)) rc >>= 1;
    if (p.n_range % rc == 0) {
      int lrc = 0;
      while ((1 << lrc) < rc) ++lrc;
      const size_t smem = doppler2_smem(L1, L2, rc);
      const dim3 grid(p.n_range / rc, p.n_chan, p.batch);
      const auto* x = reinterpret_cast<const float2*>(raw);
      auto* y = reinterpret_cast<float2*>(cube);
      auto launch = [&](auto kern) -> stap_status {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
          cudaGetLastError();
          return STAP_ERR_CUDA;
        }
        kern<<<grid, kDopplerThreads, smem, st>>>(x, window, y, p.n_chan, p.n_range, lrc, doppler2_pad(rc));
        return check_launch();
      };
      switch (D) {
        case 16: return launch(doppler2_kernel<4, 4>);
        case 32: return launch(doppler2_kernel<8, 4>);
        case 64: return launch(doppler2_kernel<8, 8>);
        case 128: return launch(doppler2_kernel<16, 8>);
        case 256: return launch(doppler2_kernel<16, 16>);
        case 512: return launch(doppler2_kernel<32, 16>);
        default: return launch(doppler2_kernel<32, 32>);
      }
    }
  }
  const int rc = doppler_rc(D, p.n_range);
  const size_t smem = doppler_smem(D, rc);
  int logD = 0, lrc = 0;
  while ((1 << logD) < D) ++logD;
  while ((1 << lrc) < rc) ++lrc;
  if (cudaFuncSetAttribute(doppler_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    return STAP_ERR_CUDA;
  }
  dim3 grid(p.n_range / rc, p.n_chan, p.batch);
  doppler_kernel<<<grid, kDopplerThreads, smem, st>>>(reinterpret_cast<const float2*>(raw), window,
                                                      reinterpret_cast<float2*>(cube), D, logD, p.n_chan,
                                                      p.n_range, lrc);
  return check_launch();
}

stap_status stap_covariance(const stap_plan* pl, const stap_c64* cube, stap_c64* cov, cudaStream_t st) {
  if (!pl || !cube || !cov) return STAP_ERR_NULL_ARG;
  if (!aligned16(cube) || !aligned16(cov)) return STAP_ERR_MISALIGNED;
  DeviceGuard g(pl->prm.device);
  if (!g.ok) return STAP_ERR_DEVICE;
  const stap_status s = cov_launch(pl, reinterpret_cast<const float2*>(cube), reinterpret_cast<float2*>(cov), st);
  if (s != STAP_OK) return s;
  return check_launch();
}

stap_status stap_solve_weights(const stap_plan* pl, const stap_c64* cov, const stap_c64* steering,
                               stap_c64* weights, float* gamma, int32_t* info, cudaStream_t st) {
  if (!pl || !cov || !steering || !weights || !info) return STAP_ERR_NULL_ARG;
  if (!aligned16(cov) || !aligned16(steering) || !aligned16(weights) || !aligned16(info) ||
      (gamma && !aligned16(gamma)))
    return STAP_ERR_MISALIGNED;
  DeviceGuard g(pl->prm.device);
  if (!g.ok) return STAP_ERR_DEVICE;
  solve_dispatch(pl, reinterpret_cast<const float2*>(cov), reinterpret_cast<const float2*>(steering),
                 reinterpret_cast<float2*>(weights), gamma, info, st);
  return check_launch();
}

stap_status stap_apply(const stap_plan* pl, const stap_c64* cube, const stap_c64* weights, stap_c64* out,
                       cudaStream_t st) {
  if (!pl || !cube || !weights || !out) return STAP_ERR_NULL_ARG;
  if (!aligned16(cube) || !aligned16(weights) || !aligned16(out)) return STAP_ERR_MISALIGNED;
  DeviceGuard g(pl->prm.device);
  if (!g.ok) return STAP_ERR_DEVICE;
  const stap_status s = apply_launch(pl, reinterpret_cast<const float2*>(cube),
                                     reinterpret_cast<const float2*>(weights), reinterpret_cast<float2*>(out), st);
  if (s != STAP_OK) return s;
  return check_launch();
}

stap_status stap_run(const stap_plan* pl, const stap_c64* cube, const stap_c64* steering, stap_c64* out,
                     int32_t* info, void* workspace, size_t workspace_bytes, cudaStream_t st) {
  if (!pl || !cube || !steering || !out || !info) return STAP_ERR_NULL_ARG;
  if (pl->ws_total && !workspace) return STAP_ERR_NULL_ARG;
  if (workspace_bytes < pl->ws_total) return STAP_ERR_BAD_DIMS;
  if (!aligned16(cube) || !aligned16(steering) || !aligned16(out) || !aligned16(info) ||
      (workspace && !aligned16(workspace)))
    return STAP_ERR_MISALIGNED;
  DeviceGuard g(pl->prm.device);
  if (!g.ok) return STAP_ERR_DEVICE;
  if (pl->fused) {
    fused_launch(pl->fcfg, pl->kp, reinterpret_cast<const float2*>(cube), reinterpret_cast<const float2*>(steering),
                 reinterpret_cast<float2*>(out), info, st);
    return check_launch();
  }
  return staged_run(pl, reinterpret_cast<const float2*>(cube), reinterpret_cast<const float2*>(steering),
                    reinterpret_cast<float2*>(out), info, workspace, st);
}

stap_status stap_run_host(const stap_plan* pl, const stap_c64* h_cube, const stap_c64* h_steering, stap_c64* h_out,
                          int32_t* h_info, void* workspace, size_t workspace_bytes, cudaStream_t st) {
  if (!pl || !h_cube || !h_steering || !h_out || !h_info || !workspace) return STAP_ERR_NULL_ARG;
  if (pl->prm.out_multicast || pl->prm.out_n_peers) return STAP_ERR_UNSUPPORTED;  // a host `out` is not a multicast address
  size_t need = 0;
  stap_plan_workspace_bytes(pl, 1, &need);
  if (workspace_bytes < need) return STAP_ERR_BAD_DIMS;
  if (!aligned16(workspace)) return STAP_ERR_MISALIGNED;
  DeviceGuard g(pl->prm.device);
  if (!g.ok) return STAP_ERR_DEVICE;
  char* w = static_cast<char*>(workspace);
  char* d_cube = w + pl->ws_total;
  char* d_steer = d_cube + align_up(pl->cube_bytes, 256);
  char* d_out = d_steer + align_up(pl->steer_bytes, 256);
  char* d_info = d_out + align_up(pl->out_bytes, 256);
  if (pl->io_nch) {
    // chunk c: H2D on io_s[0] -> kernels on `st` -> D2H on io_s[1]; PCIe runs both directions
    // at once, so the D2H of chunk c overlaps the H2D of chunk c+1 and the kernels
    const stap_plan* ch = pl->io_child;
    cudaStream_t sin = pl->io_s[0], sout = pl->io_s[1];
    cudaEvent_t e_entry = pl->io_ev[0], e_exit = pl->io_ev[1];
    const cudaEvent_t* e_in = pl->io_ev + 2;
    const cudaEvent_t* e_done = pl->io_ev + 2 + pl->io_nch;
    bool ok = cudaEventRecord(e_entry, st) == cudaSuccess && cudaStreamWaitEvent(sin, e_entry, 0) == cudaSuccess &&
              cudaStreamWaitEvent(sout, e_entry, 0) == cudaSuccess &&
              cudaMemcpyAsync(d_steer, h_steering, pl->steer_bytes, cudaMemcpyHostToDevice, sin) == cudaSuccess;
    for (int c = 0; ok && c < pl->io_nch; ++c) {
      ok = cudaMemcpyAsync(d_cube + c * ch->cube_bytes, reinterpret_cast<const char*>(h_cube) + c * ch->cube_bytes,
                           ch->cube_bytes, cudaMemcpyHostToDevice, sin) == cudaSuccess &&
           cudaEventRecord(e_in[c], sin) == cudaSuccess;
    }
    for (int c = 0; ok && c < pl->io_nch; ++c) {
      ok = cudaStreamWaitEvent(st, e_in[c], 0) == cudaSuccess &&
           stap_run(ch, reinterpret_cast<const stap_c64*>(d_cube + c * ch->cube_bytes),
                    reinterpret_cast<const stap_c64*>(d_steer), reinterpret_cast<stap_c64*>(d_out + c * ch->out_bytes),
                    reinterpret_cast<int32_t*>(d_info + c * ch->info_bytes), workspace, ch->ws_total, st) == STAP_OK &&
           cudaEventRecord(e_done[c], st) == cudaSuccess && cudaStreamWaitEvent(sout, e_done[c], 0) == cudaSuccess &&
           cudaMemcpyAsync(reinterpret_cast<char*>(h_out) + c * ch->out_bytes, d_out + c * ch->out_bytes, ch->out_bytes,
                           cudaMemcpyDeviceToHost, sout) == cudaSuccess &&
           cudaMemcpyAsync(reinterpret_cast<char*>(h_info) + c * ch->info_bytes, d_info + c * ch->info_bytes,
                           ch->info_bytes, cudaMemcpyDeviceToHost, sout) == cudaSuccess;
    }
    ok = ok && cudaEventRecord(e_exit, sout) == cudaSuccess && cudaStreamWaitEvent(st, e_exit, 0) == cudaSuccess;
    if (!ok) {
      cudaGetLastError();
      return STAP_ERR_CUDA;
    }
    return STAP_OK;
  }
  if (cudaMemcpyAsync(d_cube, h_cube, pl->cube_bytes, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaMemcpyAsync(d_steer, h_steering, pl->steer_bytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
  {
    cudaGetLastError();
    return STAP_ERR_CUDA;
  }
  stap_status s = stap_run(pl, reinterpret_cast<const stap_c64*>(d_cube), reinterpret_cast<const stap_c64*>(d_steer),
                           reinterpret_cast<stap_c64*>(d_out), reinterpret_cast<int32_t*>(d_info), workspace,
                           pl->ws_total, st);
  if (s != STAP_OK) return s;
  if (cudaMemcpyAsync(h_out, d_out, pl->out_bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(h_info, d_info, pl->info_bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess) {
    cudaGetLastError();
    return STAP_ERR_CUDA;
  }
  return STAP_OK;
}

#ifdef STAPK_PROF
// Profiling builds only: read and reset the fused kernel's phase-cycle counters.
int stap_debug_fused_prof(unsigned long long* out4) {
  cudaMemcpyFromSymbol(out4, g_fused_prof, sizeof(unsigned long long) * 4);
  unsigned long long z[4] = {0, 0, 0, 0};
  cudaMemcpyToSymbol(g_fused_prof, z, sizeof z);
  return (int)cudaGetLastError();
}
#endif

}  // extern "C"

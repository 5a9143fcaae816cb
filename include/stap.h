/*
 * include/stap.h -- C ABI of libstap.so, the B200 (sm_100a) STAP hot path.
 *
 * What the library computes (BASELINE.json north_star; the paper itself never
 * states the STAP mathematics, so every convention is a DESIGN.md "reading"):
 *
 *   datacube X[D][C][R] complex64: Doppler bins x channels x range cells, i.e.
 *     the paper's "# pulses per cube, # channels, # samples per pulse"
 *     (sec. 5.3) after the per-row Doppler FFT (PAPER.md:340,
 *     Table 2 row "fft_2D,axis=1"); readings c-1, c-14.
 *   unit (d, b): Doppler bin d, training block b = range cells [bK, bK+K)
 *     (reading c-7); units are independent -- the outer parallel loop of
 *     PAPER.md:420-430 (Fig. 7 text) and PAPER.md:408-418.
 *   snapshot z_{d,r}[t*C + c] = X[(d - h + t) mod D][c][r], h = floor((T-1)/2)
 *     (readings c-2, c-3, c-4).
 *   stap_covariance    : R_{d,b} = (1/K) sum_{r in b} z z^H + delta I,
 *                        delta = lambda tr(Rhat)/N            (c-5, c-6)
 *   stap_solve_weights : R = L L^H (Cholesky), y_k = L^-1 s_k, gamma_k = ||y_k||^2,
 *                        w_k = L^-H y_k / gamma_k  (MVDR, w_k^H s_k = 1)  (c-9, c-10)
 *   stap_apply         : Y[d][k][r] = w_{d,b(r),k}^H z_{d,r}     (c-12)
 *   stap_run           : all of the above, fused, cube in -> Y out.
 *
 * Conventions (all entry points):
 *  - Layouts are row-major, last index fastest.  complex64 = {float re, im}
 *    interleaved (== torch.complex64 == cuFloatComplex).
 *  - Device pointers must be 16-byte aligned device memory of the plan's
 *    device; the caller owns every buffer; inputs are const and never written.
 *  - Every call only enqueues work on `stream` and returns (no host sync, no
 *    allocation), so calls are CUDA-graph capturable -- except stap_run_host,
 *    which also enqueues the host<->device copies.  Argument errors are
 *    returned synchronously and NOTHING is launched.  Numerical failures are
 *    reported on the device in `info` (reading c-11):
 *        0       the unit is fine
 *        j > 0   Cholesky pivot j (1-based) was <= 0 or not finite: every
 *                weight and output of that unit is 0
 *        -(k+1)  gamma_k <= 0 or not finite for the smallest such k: the
 *                weights/outputs of every failing k are 0.
 *  - Arithmetic: complex64 in and out, FP32 FFMA throughout under the default
 *    stap_params.precision = STAP_PREC_FP32 (no TF32, no fast-math; the solver's
 *    1/pivot is the hardware reciprocal, rcp.approx, ~1 ulp).  STAP_PREC_TF32X3 opts
 *    the covariance (24 <= N <= 64, K % 16 == 0) and the weight application (S == 16,
 *    K % 64 == 0) into tcgen05 tensor-core MMAs in 3xTF32 (each FP32 operand split
 *    hi + lo, hi*hi + hi*lo + lo*hi, FP32 accumulation; measured per-R error
 *    <= 2.3e-6, per-Y-line <= 5e-7 against the fp64 oracle); which kernels a plan
 *    runs is fixed at plan creation (stap_plan_describe) and never changes per call.
 *    Results match the fp64 oracle to the tolerances in DESIGN.md, not bitwise.  A
 *    given plan computes every unit with a fixed summation order that does not depend
 *    on dop_begin, dop_count or batch: shards are bitwise identical to the unsharded run.
 *  - There is no CPU fallback: without an sm_100 device every call fails.
 */
#ifndef STAP_H_
#define STAP_H_

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STAP_ABI_VERSION 4

typedef struct { float re, im; } stap_c64;
typedef struct stap_plan stap_plan;

typedef enum {
    STAP_OK = 0,
    STAP_ERR_NULL_ARG = 1,     /* a required pointer is NULL */
    STAP_ERR_BAD_DIMS = 2,     /* a dim <= 0, R % K != 0, T > D, shard or cube window
                                  out of range, lambda < 0 or not finite, workspace too small */
    STAP_ERR_UNSUPPORTED = 3,  /* valid but not implemented: N = C*T > 64, S > 32, K odd,
                                  K > 1024, C > 8 */
    STAP_ERR_MISALIGNED = 4,   /* a device pointer is not 16-byte aligned */
    STAP_ERR_CUDA = 5,         /* a CUDA runtime / launch error (incl. a tensor map that cannot be
                                  encoded for the given cube pointer) */
    STAP_ERR_NCCL = 6,         /* multi-GPU extension: NCCL missing, or an NCCL / IPC call failed */
    STAP_ERR_DEVICE = 7        /* no device, or the plan's device is not sm_100 */
} stap_status;

typedef struct {
    int32_t n_chan;          /* C  channels                      ("# channels") */
    int32_t tdof;            /* T  temporal DOF: adjacent Doppler bins per snapshot (north_star) */
    int32_t n_dop;           /* D  Doppler bins, global          ("# pulses per cube") */
    int32_t n_range;         /* R  range cells                   ("# samples per pulse") */
    int32_t training_block;  /* K  range cells per training block; R % K == 0 (north_star) */
    int32_t n_steering;      /* S  steering vectors              (north_star) */
    float   diag_load;       /* lambda >= 0, delta = lambda tr(Rhat)/N (reading c-6) */
    int32_t dop_begin;       /* first owned Doppler bin (0 on one GPU)                    */
    int32_t dop_count;       /* owned bins D_loc (n_dop on one GPU)                        */
    int32_t cube_bin0;       /* global bin held in row 0 of the cube buffer               */
    int32_t cube_bins;       /* bins held by the cube buffer (n_dop = the whole cube); the
                                buffer holds bins cube_bin0 .. cube_bin0+cube_bins-1 mod D
                                and must cover every owned bin's window                   */
    int32_t batch;           /* independent cubes per call (>= 1), stored back to back     */
    int32_t device;          /* CUDA ordinal the plan launches on                          */
    int32_t path;            /* stap_run's kernel path, a stap_path value (0 = auto)       */
    int32_t out_multicast;   /* ABI v3.  0: `out` of stap_apply / stap_run is an ordinary
                                device pointer (own memory or a peer-mapped buffer).
                                1: `out` is an NVLS multicast address (CUDA multicast object
                                bound to every rank's copy of the output buffer, e.g. torch
                                symmetric memory's multicast_ptr plus this rank's offset);
                                every Y store is a multimem.st, so each rank's kernels write
                                their outputs into all ranks' buffers (an all-gather inside
                                the apply epilogue).  The caller orders
                                the stores before reading (a cross-rank barrier after the
                                stream's work).  stap_run_host rejects 1 (host `out`)
                                with STAP_ERR_UNSUPPORTED; any other value is
                                STAP_ERR_BAD_DIMS.                                         */
    int32_t out_n_peers;     /* ABI v3.  0..7 (else STAP_ERR_BAD_DIMS; > 0 together with
                                out_multicast is STAP_ERR_BAD_DIMS).  Every Y store to `out`
                                is repeated at out + out_peer_offset[i] (bytes), i < out_n_peers:
                                peer-mapped copies of the same output slice in the other
                                ranks' buffers (e.g. torch symmetric memory's get_buffer), so
                                the apply epilogue performs an all-gather by unicast stores
                                over NVLink.  Offsets must be multiples of 16
                                (else STAP_ERR_MISALIGNED); the caller guarantees each
                                out + offset range is mapped and writable.  stap_run_host
                                rejects out_n_peers > 0 with STAP_ERR_UNSUPPORTED.           */
    int64_t out_peer_offset[7];
    int32_t precision;       /* ABI v4.  A stap_precision value (0 = STAP_PREC_FP32, the default;
                                else STAP_ERR_BAD_DIMS)                                    */
} stap_params;

/* Arithmetic of the covariance and apply stages (include/stap.h header "Arithmetic").
 * STAP_PREC_FP32: FP32 FFMA everywhere.  STAP_PREC_TF32X3: tcgen05 3xTF32 covariance and
 * apply where the shape allows (see above), FP32 elsewhere; opt-in only. */
typedef enum { STAP_PREC_FP32 = 0, STAP_PREC_TF32X3 = 1 } stap_precision;

/* stap_run path.  AUTO picks the measured-faster one: the staged path when both its
 * tensor-core stages are in use (precision = STAP_PREC_TF32X3 and covariance:
 * 24 <= N <= 64, K % 16 == 0; apply: S = 16, K % 64 == 0, N <= 64 -- medium, large), else
 * the fused kernel when the shape fits it (small, medium), else staged.  FUSED on a shape the fused kernel cannot hold is
 * STAP_ERR_UNSUPPORTED.  The stage entry points are independent of this field. */
typedef enum { STAP_PATH_AUTO = 0, STAP_PATH_FUSED = 1, STAP_PATH_STAGED = 2 } stap_path;

/* Buffer shapes (complex64 unless noted), with B = R/K, N = C*T, Dl = dop_count:
 *   cube     [batch][cube_bins][C][R]
 *   steering [S][N]                    (element i = t*C + c; shared by every unit)
 *   cov      [batch][Dl][B][N][N]      (full Hermitian, loading applied)
 *   weights  [batch][Dl][B][S][N]
 *   gamma    [batch][Dl][B][S]   float (nullable)
 *   info     [batch][Dl][B]      int32
 *   out      [batch][Dl][S][R]     (Doppler-major: shard g starts at dop_begin*S*R) */

/* Validate `p` and build an immutable plan (host metadata only). */
stap_status stap_plan_create(const stap_params* p, stap_plan** out_plan);
/* Legal once all work using the plan has completed. NULL is accepted. */
stap_status stap_plan_destroy(stap_plan* plan);
/* Device workspace stap_run (host_io = 0) or stap_run_host (host_io = 1) needs. */
stap_status stap_plan_workspace_bytes(const stap_plan* plan, int32_t host_io, size_t* bytes);
/* Kernel the plan selected for stap_run ("fused:..." or "staged:..."), for logs. */
const char* stap_plan_describe(const stap_plan* plan);

/* Stage 1: loaded covariance of every owned unit.  Reads only the bins each window needs. */
stap_status stap_covariance(const stap_plan* plan, const stap_c64* cube, stap_c64* cov,
                            cudaStream_t stream);
/* Front end (DESIGN reading c-19): the datacube from raw pulses,
 *   cube[n][d][c][r] = sum_{p < D} window[p] raw[n][p][c][r] exp(-2 pi i p d / D),
 * the per-row taper and FFT along the pulse axis (Table 2 "fft_2D,axis=1").
 * raw and cube: [batch][D][C][R] complex64 (device, 16-byte aligned, distinct);
 * window: D floats (device).  Needs a plan over the whole cube (dop_begin = 0,
 * dop_count = cube_bins = n_dop, cube_bin0 = 0) and D a power of two, 2 <= D <= 8192:
 * otherwise STAP_ERR_UNSUPPORTED. */
stap_status stap_doppler(const stap_plan* plan, const float* window, const stap_c64* raw, stap_c64* cube,
                         cudaStream_t stream);
/* Stage 2: Cholesky + forward/back solves -> MVDR weights, gamma, info. */
stap_status stap_solve_weights(const stap_plan* plan, const stap_c64* cov, const stap_c64* steering,
                               stap_c64* weights, float* gamma, int32_t* info, cudaStream_t stream);
/* Stage 3: Y = W^H z for every owned bin and range cell. */
stap_status stap_apply(const stap_plan* plan, const stap_c64* cube, const stap_c64* weights,
                       stap_c64* out, cudaStream_t stream);
/* Whole path.  `workspace` (device, >= stap_plan_workspace_bytes(plan, 0, .) bytes,
 * may be NULL when that is 0) holds intermediates when the plan is staged. */
stap_status stap_run(const stap_plan* plan, const stap_c64* cube, const stap_c64* steering,
                     stap_c64* out, int32_t* info, void* workspace, size_t workspace_bytes,
                     cudaStream_t stream);
/* Whole path from HOST buffers (pinned for async copies): enqueues H2D of cube and
 * steering, the kernels, and D2H of out and info; the caller synchronises `stream`
 * before reading h_out / h_info (the call makes `stream` wait for everything it
 * enqueued).  For batch >= 2 the plan pipelines the batch in up to 8 chunks of whole
 * cubes on two internal streams (H2D of chunk c+1 and D2H of chunk c-1 overlap the
 * kernels of chunk c; PCIe moves both directions at once); calls on one plan must
 * therefore come from one host thread at a time.  Device staging lives in
 * `workspace` (>= stap_plan_workspace_bytes(plan, 1, .)). */
stap_status stap_run_host(const stap_plan* plan, const stap_c64* h_cube, const stap_c64* h_steering,
                          stap_c64* h_out, int32_t* h_info, void* workspace, size_t workspace_bytes,
                          cudaStream_t stream);

const char* stap_status_string(stap_status s);
int32_t stap_abi_version(void);

/* ---- Multi-GPU extension.  Doppler bins shard over ranks with no
 * data-path exchange (each rank's plan owns dop_begin .. dop_begin+dop_count-1, its cube
 * buffer holds those bins plus the T-1 halo); the only collective is the OPTIONAL gather of
 * the Doppler-major outputs -- the analogue of the paper's per-chunk result return
 * (the pfor driver reassembling per-chunk slices).
 *
 * The gathered buffer of every rank, out_full, is [nranks][batch][Dl][S][R] complex64 (for
 * batch = 1 and equal shards that is the global Doppler-major [D][S][R]); rank r's plan
 * writes its own slice, out_full + r*batch*Dl*S*R.  NCCL (2.x, libnccl.so.2) is loaded at
 * run time on the first stap_comm call; without it the calls return STAP_ERR_NCCL and the
 * single-GPU library is unaffected.  A communicator is used from one host thread at a time. */
typedef struct stap_comm stap_comm;
/* 128 bytes that name a new communicator; produced on one rank, handed to all (any channel). */
stap_status stap_comm_unique_id(uint8_t id[128]);
/* One process driving `ndev` GPUs (ranks 0..ndev-1 = devices[0..ndev-1]): an NCCL clique
 * (ncclCommInitAll) plus peer access between every pair of devices. */
stap_status stap_comm_create(int32_t ndev, const int32_t* devices, stap_comm** out_comm);
/* One process per GPU: this process's rank `rank` of `nranks`, on CUDA ordinal `device`. */
stap_status stap_comm_init_rank(int32_t nranks, int32_t rank, const uint8_t id[128], int32_t device,
                                stap_comm** out_comm);
/* Ranks in the communicator and devices driven by this process (1 under init_rank). */
stap_status stap_comm_size(const stap_comm* comm, int32_t* nranks, int32_t* nlocal);
/* In-place all-gather of the outputs (ncclAllGather, one group call): for every local device
 * i, out_full[i] (device memory of that device, layout above) and plans[i] (that rank's plan:
 * the same batch, dop_count, S and R on every rank, else STAP_ERR_BAD_DIMS); enqueued on
 * streams[i], after which every rank's out_full holds every rank's slice. */
stap_status stap_comm_allgather_out(stap_comm* comm, stap_c64* const* out_full, const stap_plan* const* plans,
                                    const cudaStream_t* streams);
/* The all-gather fused into the apply epilogue: writes, for every local
 * device i, offsets[i*7 + 0 .. n_peers-1] = the byte offsets from this rank's slice of
 * out_full[i] to the same slice of every other rank's out_full (peer memory: peer access in one
 * process; CUDA IPC over the NCCL communicator across processes -- out_full must then be a
 * cudaMalloc allocation or lie inside one).  Passing them as stap_params.out_n_peers /
 * out_peer_offset makes every Y store of stap_run / stap_apply land in every rank's buffer; the
 * caller orders the stores before reading (stream sync + a barrier across ranks).  Collective:
 * every rank calls it with its own buffers; a repeat call with the buffers of the previous call
 * returns the same offsets without communicating (peers stay mapped until stap_comm_destroy).
 * n_peers = nranks - 1 <= 7. */
stap_status stap_comm_peer_offsets(stap_comm* comm, stap_c64* const* out_full, int64_t* offsets, int32_t* n_peers);
/* The gather by copy engines: for every local device i, one peer copy of this rank's slice of
 * out_full[i] into every other rank's out_full (cudaMemcpyAsync over NVLink, each peer's copy
 * on its own internal stream -- its own copy engine -- forked from and joined back into
 * streams[i]; no SM time, so it overlaps the next step's kernels when streams[i] is not the
 * compute stream).  Needs a prior stap_comm_peer_offsets on the same out_full (the peer
 * mapping), else STAP_ERR_BAD_DIMS; plans as in stap_comm_allgather_out.  The caller orders
 * the copies before reading (stream sync + a barrier across ranks). */
stap_status stap_comm_push_out(stap_comm* comm, stap_c64* const* out_full, const stap_plan* const* plans,
                               const cudaStream_t* streams);
/* Frees the NCCL communicators and closes the IPC mappings; NULL is accepted. */
stap_status stap_comm_destroy(stap_comm* comm);

#ifdef __cplusplus
}
#endif
#endif /* STAP_H_ */

// comm.cu -- the multi-GPU extension of the C ABI (include/stap.h "Multi-GPU extension"):
// NCCL communicators over the ranks' Doppler-bin shards, the optional in-place all-gather of
// the Doppler-major outputs, and the peer offsets that fuse that gather into the apply
// epilogue (the paper's per-chunk result return,
// PAPER.md:447-463, 648-654).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, the copy already loaded by the host
// process if any -- e.g. torch's), so libstap.so has no link dependency on it and the
// single-GPU entry points never need it.  Nothing here does arithmetic of the method.
#include <dlfcn.h>

#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include "internal.h"

namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's copy, if loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.CommInitAll = reinterpret_cast<decltype(a.CommInitAll)>(dlsym(h, "ncclCommInitAll"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(h, "ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.GetUniqueId && a.CommInitAll && a.CommInitRank && a.CommDestroy && a.AllGather && a.GroupStart &&
           a.GroupEnd && a.GetErrorString;
    return a;
  }();
  return api;
}

bool nccl_ok(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return true;
  fprintf(stderr, "libstap: %s failed: %s\n", what, nccl().GetErrorString(r));
  return false;
}

// cuMemGetAddressRange from the driver (base of the allocation holding a pointer), no libcuda link
using PFN_range = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
PFN_range mem_range_fn() {
  static PFN_range fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_range>(f);
  }();
  return fn;
}

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int d) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != d) cudaSetDevice(d);
  }
  ~DevGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// what one rank publishes so that the others can map its output buffer
struct IpcRecord {
  cudaIpcMemHandle_t handle;
  uint64_t offset;  // of out_full inside the allocation
  uint64_t pad;
};

}  // namespace

struct stap_comm {
  int nranks = 0, nlocal = 0;
  std::vector<int> devices, ranks;
  std::vector<ncclComm_t> comms;
  std::vector<void*> ipc_opened;  // peer allocations mapped by stap_comm_peer_offsets (closed at destroy)
  int ipc_device = -1;
  // recorded by stap_comm_peer_offsets: per local device i, its out_full and every rank's
  // out_full as addressable from this process (own rank: out_full[i] itself)
  std::vector<char*> mapped_out;
  std::vector<std::vector<char*>> peer_full;
  // stap_comm_push_out's fork-join: per local device, one stream per peer (the copies to
  // different peers run on different copy engines) and the events that chain them
  std::vector<std::vector<cudaStream_t>> push_streams;
  std::vector<cudaEvent_t> push_fork;
  std::vector<std::vector<cudaEvent_t>> push_join;
};

extern "C" {

stap_status stap_comm_unique_id(uint8_t id[128]) {
  if (!id) return STAP_ERR_NULL_ARG;
  if (!nccl().ok) return STAP_ERR_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  ncclUniqueId u;
  if (!nccl_ok(nccl().GetUniqueId(&u), "ncclGetUniqueId")) return STAP_ERR_NCCL;
  memcpy(id, &u, 128);
  return STAP_OK;
}

stap_status stap_comm_create(int32_t ndev, const int32_t* devices, stap_comm** out_comm) {
  if (!devices || !out_comm) return STAP_ERR_NULL_ARG;
  *out_comm = nullptr;
  if (ndev < 1 || ndev > 8) return STAP_ERR_BAD_DIMS;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) {
    cudaGetLastError();
    return STAP_ERR_DEVICE;
  }
  for (int i = 0; i < ndev; ++i) {
    if (devices[i] < 0 || devices[i] >= count) return STAP_ERR_DEVICE;
    for (int j = 0; j < i; ++j)
      if (devices[j] == devices[i]) return STAP_ERR_BAD_DIMS;
  }
  if (!nccl().ok) return STAP_ERR_NCCL;
  stap_comm* c = new (std::nothrow) stap_comm();
  if (!c) return STAP_ERR_CUDA;
  c->nranks = c->nlocal = ndev;
  c->devices.assign(devices, devices + ndev);
  for (int i = 0; i < ndev; ++i) c->ranks.push_back(i);
  c->comms.assign(ndev, nullptr);
  if (!nccl_ok(nccl().CommInitAll(c->comms.data(), ndev, devices), "ncclCommInitAll")) {
    delete c;
    return STAP_ERR_NCCL;
  }
  // peer access between every pair (the fused gather's stores go straight to peer memory)
  for (int i = 0; i < ndev; ++i) {
    DevGuard g(devices[i]);
    for (int j = 0; j < ndev; ++j) {
      if (i == j) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, devices[i], devices[j]);
      if (can) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
          cudaGetLastError();
          stap_comm_destroy(c);
          return STAP_ERR_CUDA;
        }
        cudaGetLastError();
      }
    }
  }
  *out_comm = c;
  return STAP_OK;
}

stap_status stap_comm_init_rank(int32_t nranks, int32_t rank, const uint8_t id[128], int32_t device,
                                stap_comm** out_comm) {
  if (!id || !out_comm) return STAP_ERR_NULL_ARG;
  *out_comm = nullptr;
  if (nranks < 1 || nranks > 8 || rank < 0 || rank >= nranks) return STAP_ERR_BAD_DIMS;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) {
    cudaGetLastError();
    return STAP_ERR_DEVICE;
  }
  if (!nccl().ok) return STAP_ERR_NCCL;
  stap_comm* c = new (std::nothrow) stap_comm();
  if (!c) return STAP_ERR_CUDA;
  c->nranks = nranks;
  c->nlocal = 1;
  c->devices = {device};
  c->ranks = {rank};
  c->comms.assign(1, nullptr);
  ncclUniqueId u;
  memcpy(&u, id, 128);
  DevGuard g(device);
  if (!nccl_ok(nccl().CommInitRank(&c->comms[0], nranks, u, rank), "ncclCommInitRank")) {
    delete c;
    return STAP_ERR_NCCL;
  }
  *out_comm = c;
  return STAP_OK;
}

stap_status stap_comm_size(const stap_comm* c, int32_t* nranks, int32_t* nlocal) {
  if (!c || !nranks || !nlocal) return STAP_ERR_NULL_ARG;
  *nranks = c->nranks;
  *nlocal = c->nlocal;
  return STAP_OK;
}

// every local plan describes the same output slice shape; returns its bytes (0 on a mismatch)
static size_t slice_bytes(const stap_comm* c, const stap_plan* const* plans) {
  size_t bytes = 0;
  stapk::PlanOutGeom g0{};
  for (int i = 0; i < c->nlocal; ++i) {
    stapk::PlanOutGeom g;
    if (!plans[i] || !stapk::plan_out_geom(plans[i], &g)) return 0;
    if (g.device != c->devices[i]) return 0;
    if (i == 0) {
      g0 = g;
      bytes = g.out_bytes;
    } else if (g.batch != g0.batch || g.dop_count != g0.dop_count || g.S != g0.S || g.R != g0.R) {
      return 0;
    }
  }
  return bytes;
}

stap_status stap_comm_allgather_out(stap_comm* c, stap_c64* const* out_full, const stap_plan* const* plans,
                                    const cudaStream_t* streams) {
  if (!c || !out_full || !plans || !streams) return STAP_ERR_NULL_ARG;
  for (int i = 0; i < c->nlocal; ++i)
    if (!out_full[i] || !plans[i]) return STAP_ERR_NULL_ARG;
  const size_t bytes = slice_bytes(c, plans);
  if (!bytes || bytes % 4) return STAP_ERR_BAD_DIMS;
  for (int i = 0; i < c->nlocal; ++i)
    if (reinterpret_cast<uintptr_t>(out_full[i]) & 15u) return STAP_ERR_MISALIGNED;
  const size_t count = bytes / 4;  // floats per rank slice
  const NcclApi& n = nccl();
  if (!nccl_ok(n.GroupStart(), "ncclGroupStart")) return STAP_ERR_NCCL;
  bool ok = true;
  for (int i = 0; i < c->nlocal && ok; ++i) {
    char* base = reinterpret_cast<char*>(out_full[i]);
    ok = nccl_ok(n.AllGather(base + (size_t)c->ranks[i] * bytes, base, count, ncclFloat32, c->comms[i], streams[i]),
                 "ncclAllGather");
  }
  const bool ended = nccl_ok(n.GroupEnd(), "ncclGroupEnd");
  return ok && ended ? STAP_OK : STAP_ERR_NCCL;
}

stap_status stap_comm_peer_offsets(stap_comm* c, stap_c64* const* out_full, int64_t* offsets, int32_t* n_peers) {
  if (!c || !out_full || !offsets || !n_peers) return STAP_ERR_NULL_ARG;
  if (c->nranks - 1 > 7) return STAP_ERR_UNSUPPORTED;
  for (int i = 0; i < c->nlocal; ++i) {
    if (!out_full[i]) return STAP_ERR_NULL_ARG;
    if (reinterpret_cast<uintptr_t>(out_full[i]) & 15u) return STAP_ERR_MISALIGNED;
  }
  *n_peers = c->nranks - 1;
  // the same buffers again: the peers are mapped already (an IPC handle opens once per process)
  bool same = (int)c->mapped_out.size() == c->nlocal;
  for (int i = 0; i < c->nlocal && same; ++i) same = c->mapped_out[i] == reinterpret_cast<char*>(out_full[i]);
  if (same) {
    for (int i = 0; i < c->nlocal; ++i) {
      int k = 0;
      for (int j = 0; j < c->nranks; ++j)
        if (j != c->ranks[i]) offsets[i * 7 + k++] = c->peer_full[i][j] - c->mapped_out[i];
      for (; k < 7; ++k) offsets[i * 7 + k] = 0;
    }
    return STAP_OK;
  }
  c->mapped_out.clear();  // set again only once every peer is mapped (stap_comm_push_out checks it)
  c->peer_full.assign(c->nlocal, std::vector<char*>(c->nranks, nullptr));
  if (c->nlocal == c->nranks) {
    // one process: every buffer is addressable from every device (peer access, unified VA)
    for (int i = 0; i < c->nlocal; ++i) {
      int k = 0;
      for (int j = 0; j < c->nranks; ++j) {
        c->peer_full[i][j] = reinterpret_cast<char*>(out_full[j]);
        if (j != i)
          offsets[i * 7 + k++] = reinterpret_cast<char*>(out_full[j]) - reinterpret_cast<char*>(out_full[i]);
      }
      for (; k < 7; ++k) offsets[i * 7 + k] = 0;
    }
    c->mapped_out.assign(reinterpret_cast<char* const*>(out_full), reinterpret_cast<char* const*>(out_full) + c->nlocal);
    return STAP_OK;
  }
  // one process per GPU: publish (IPC handle of the allocation, offset) through the
  // communicator, map every peer's allocation here
  if (c->nlocal != 1) return STAP_ERR_UNSUPPORTED;
  const PFN_range range = mem_range_fn();
  if (!range) return STAP_ERR_CUDA;
  DevGuard g(c->devices[0]);
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(out_full[0])) != CUDA_SUCCESS) return STAP_ERR_CUDA;
  IpcRecord mine{};
  if (cudaIpcGetMemHandle(&mine.handle, reinterpret_cast<void*>(base)) != cudaSuccess) {
    cudaGetLastError();
    return STAP_ERR_CUDA;
  }
  mine.offset = reinterpret_cast<uint64_t>(out_full[0]) - (uint64_t)base;
  const size_t rec = sizeof(IpcRecord);
  static_assert(sizeof(IpcRecord) % 4 == 0, "whole floats");
  void* dbuf = nullptr;
  if (cudaMalloc(&dbuf, rec * (c->nranks + 1)) != cudaSuccess) {
    cudaGetLastError();
    return STAP_ERR_CUDA;
  }
  std::vector<IpcRecord> all(c->nranks);
  cudaStream_t st = nullptr;
  bool ok = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess;
  char* recv = static_cast<char*>(dbuf);
  char* send = recv + rec * c->nranks;
  ok = ok && cudaMemcpyAsync(send, &mine, rec, cudaMemcpyHostToDevice, st) == cudaSuccess;
  ok = ok && nccl_ok(nccl().AllGather(send, recv, rec / 4, ncclFloat32, c->comms[0], st), "ncclAllGather");
  ok = ok && cudaMemcpyAsync(all.data(), recv, rec * c->nranks, cudaMemcpyDeviceToHost, st) == cudaSuccess;
  ok = ok && cudaStreamSynchronize(st) == cudaSuccess;
  if (st) cudaStreamDestroy(st);
  cudaFree(dbuf);
  if (!ok) {
    cudaGetLastError();
    return STAP_ERR_NCCL;
  }
  int k = 0;
  c->peer_full[0][c->ranks[0]] = reinterpret_cast<char*>(out_full[0]);
  for (int j = 0; j < c->nranks; ++j) {
    if (j == c->ranks[0]) continue;
    void* peer = nullptr;
    if (cudaIpcOpenMemHandle(&peer, all[j].handle, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      return STAP_ERR_CUDA;
    }
    c->ipc_opened.push_back(peer);
    c->ipc_device = c->devices[0];
    c->peer_full[0][j] = static_cast<char*>(peer) + all[j].offset;
    offsets[k++] = c->peer_full[0][j] - reinterpret_cast<char*>(out_full[0]);
  }
  for (; k < 7; ++k) offsets[k] = 0;
  c->mapped_out.assign(1, reinterpret_cast<char*>(out_full[0]));
  return STAP_OK;
}

stap_status stap_comm_push_out(stap_comm* c, stap_c64* const* out_full, const stap_plan* const* plans,
                               const cudaStream_t* streams) {
  if (!c || !out_full || !plans || !streams) return STAP_ERR_NULL_ARG;
  const size_t bytes = slice_bytes(c, plans);
  if (!bytes) return STAP_ERR_BAD_DIMS;
  if ((int)c->mapped_out.size() != c->nlocal) return STAP_ERR_BAD_DIMS;  // no stap_comm_peer_offsets yet
  for (int i = 0; i < c->nlocal; ++i)
    if (reinterpret_cast<char*>(out_full[i]) != c->mapped_out[i]) return STAP_ERR_BAD_DIMS;
  if (c->push_streams.empty()) {  // created once per communicator
    c->push_streams.assign(c->nlocal, std::vector<cudaStream_t>(c->nranks, nullptr));
    c->push_join.assign(c->nlocal, std::vector<cudaEvent_t>(c->nranks, nullptr));
    c->push_fork.assign(c->nlocal, nullptr);
    for (int i = 0; i < c->nlocal; ++i) {
      DevGuard g(c->devices[i]);
      bool ok = cudaEventCreateWithFlags(&c->push_fork[i], cudaEventDisableTiming) == cudaSuccess;
      for (int j = 0; j < c->nranks && ok; ++j) {
        if (j == c->ranks[i]) continue;
        ok = cudaStreamCreateWithFlags(&c->push_streams[i][j], cudaStreamNonBlocking) == cudaSuccess &&
             cudaEventCreateWithFlags(&c->push_join[i][j], cudaEventDisableTiming) == cudaSuccess;
      }
      if (!ok) {
        cudaGetLastError();
        return STAP_ERR_CUDA;
      }
    }
  }
  // fork: every peer copy waits for the caller's stream, runs on its own stream (its own copy
  // engine), and the caller's stream waits for all of them (join)
  for (int i = 0; i < c->nlocal; ++i) {
    DevGuard g(c->devices[i]);
    const size_t off = (size_t)c->ranks[i] * bytes;
    bool ok = cudaEventRecord(c->push_fork[i], streams[i]) == cudaSuccess;
    for (int j = 0; j < c->nranks && ok; ++j) {
      if (j == c->ranks[i]) continue;
      cudaStream_t q = c->push_streams[i][j];
      ok = cudaStreamWaitEvent(q, c->push_fork[i], 0) == cudaSuccess &&
           cudaMemcpyAsync(c->peer_full[i][j] + off, c->mapped_out[i] + off, bytes, cudaMemcpyDefault, q) ==
               cudaSuccess &&
           cudaEventRecord(c->push_join[i][j], q) == cudaSuccess &&
           cudaStreamWaitEvent(streams[i], c->push_join[i][j], 0) == cudaSuccess;
    }
    if (!ok) {
      cudaGetLastError();
      return STAP_ERR_CUDA;
    }
  }
  return STAP_OK;
}

stap_status stap_comm_destroy(stap_comm* c) {
  if (!c) return STAP_OK;
  for (size_t i = 0; i < c->push_streams.size(); ++i) {
    DevGuard g(c->devices[i]);
    for (cudaStream_t q : c->push_streams[i])
      if (q) cudaStreamDestroy(q);
    for (cudaEvent_t e : c->push_join[i])
      if (e) cudaEventDestroy(e);
    if (c->push_fork[i]) cudaEventDestroy(c->push_fork[i]);
  }
  if (!c->ipc_opened.empty()) {
    DevGuard g(c->ipc_device);
    for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  }
  if (nccl().ok)
    for (ncclComm_t m : c->comms)
      if (m) nccl().CommDestroy(m);
  delete c;
  return STAP_OK;
}

}  // extern "C"

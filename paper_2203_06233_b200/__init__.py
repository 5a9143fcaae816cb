"""paper_2203_06233_b200 -- B200-native STAP hot path (arXiv 2203.06233, sec. 5.3).

A thin ctypes binding over ``libstap.so`` (include/stap.h).  Every step of the
path -- covariance with diagonal loading, Cholesky + forward/back solves giving
the MVDR weights, and weight application -- runs in the library's sm_100a
kernels; this module only marshals arguments (torch tensors supply device
memory and streams).  There is no CPU fallback: importing the package fails
loudly if the extension has not been built.

Entry points mirror the C ABI names: ``stap_plan_create``, ``stap_covariance``,
``stap_solve_weights``, ``stap_apply``, ``stap_run``, ``stap_run_host``,
``stap_plan_workspace_bytes``; ``StapPlan`` wraps them with shape checks.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("STAP_LIB") or os.path.join(_HERE, "libstap.so")  # STAP_LIB: profiling builds

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA extension first "
        "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)

STATUS = {0: "STAP_OK", 1: "STAP_ERR_NULL_ARG", 2: "STAP_ERR_BAD_DIMS", 3: "STAP_ERR_UNSUPPORTED",
          4: "STAP_ERR_MISALIGNED", 5: "STAP_ERR_CUDA", 6: "STAP_ERR_NCCL", 7: "STAP_ERR_DEVICE"}

SYMBOLS = ("stap_plan_create", "stap_plan_destroy", "stap_plan_workspace_bytes", "stap_plan_describe",
           "stap_doppler", "stap_covariance", "stap_solve_weights", "stap_apply", "stap_run", "stap_run_host",
           "stap_status_string", "stap_abi_version",
           "stap_comm_unique_id", "stap_comm_create", "stap_comm_init_rank", "stap_comm_size",
           "stap_comm_allgather_out", "stap_comm_peer_offsets", "stap_comm_push_out", "stap_comm_destroy")


class StapError(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        msg = _lib.stap_status_string(code).decode()
        super().__init__(f"{what}: {msg}")


PATHS = {"auto": 0, "fused": 1, "staged": 2}  # stap_path (include/stap.h)
PRECISIONS = {"fp32": 0, "tf32x3": 1}          # stap_precision (include/stap.h)


class stap_params(ctypes.Structure):
    _fields_ = [
        ("n_chan", ctypes.c_int32), ("tdof", ctypes.c_int32), ("n_dop", ctypes.c_int32),
        ("n_range", ctypes.c_int32), ("training_block", ctypes.c_int32), ("n_steering", ctypes.c_int32),
        ("diag_load", ctypes.c_float), ("dop_begin", ctypes.c_int32), ("dop_count", ctypes.c_int32),
        ("cube_bin0", ctypes.c_int32), ("cube_bins", ctypes.c_int32), ("batch", ctypes.c_int32),
        ("device", ctypes.c_int32), ("path", ctypes.c_int32), ("out_multicast", ctypes.c_int32),
        ("out_n_peers", ctypes.c_int32), ("out_peer_offset", ctypes.c_int64 * 7),
        ("precision", ctypes.c_int32),
    ]


_vp = ctypes.c_void_p
_P = ctypes.POINTER(stap_params)
_lib.stap_plan_create.argtypes = [_P, ctypes.POINTER(_vp)]
_lib.stap_plan_destroy.argtypes = [_vp]
_lib.stap_plan_workspace_bytes.argtypes = [_vp, ctypes.c_int32, ctypes.POINTER(ctypes.c_size_t)]
_lib.stap_plan_describe.argtypes = [_vp]
_lib.stap_plan_describe.restype = ctypes.c_char_p
_lib.stap_covariance.argtypes = [_vp, _vp, _vp, _vp]
_lib.stap_doppler.argtypes = [_vp, _vp, _vp, _vp, _vp]
_lib.stap_solve_weights.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp]
_lib.stap_apply.argtypes = [_vp, _vp, _vp, _vp, _vp]
_lib.stap_run.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp]
_lib.stap_run_host.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp]
_lib.stap_status_string.argtypes = [ctypes.c_int]
_lib.stap_status_string.restype = ctypes.c_char_p
_lib.stap_abi_version.restype = ctypes.c_int32
_lib.stap_comm_unique_id.argtypes = [ctypes.c_char_p]
_lib.stap_comm_create.argtypes = [ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(_vp)]
_lib.stap_comm_init_rank.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_char_p, ctypes.c_int32,
                                     ctypes.POINTER(_vp)]
_lib.stap_comm_size.argtypes = [_vp, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
_lib.stap_comm_allgather_out.argtypes = [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp)]
_lib.stap_comm_peer_offsets.argtypes = [_vp, ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_int64),
                                        ctypes.POINTER(ctypes.c_int32)]
_lib.stap_comm_push_out.argtypes = [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp)]
_lib.stap_comm_destroy.argtypes = [_vp]
for _f in ("stap_plan_create", "stap_plan_destroy", "stap_plan_workspace_bytes", "stap_doppler", "stap_covariance",
           "stap_solve_weights", "stap_apply", "stap_run", "stap_run_host", "stap_comm_unique_id",
           "stap_comm_create", "stap_comm_init_rank", "stap_comm_size", "stap_comm_allgather_out",
           "stap_comm_peer_offsets", "stap_comm_push_out", "stap_comm_destroy"):
    getattr(_lib, _f).restype = ctypes.c_int


def _check(rc: int, what: str):
    if rc != 0:
        raise StapError(rc, what)


def _ptr(t) -> _vp:
    """Raw C-ABI mirrors take torch tensors, None (NULL) or an int device address."""
    if t is None:
        return _vp(0)
    if isinstance(t, int):
        return _vp(t)
    return _vp(t.data_ptr())


def _stream(stream, device: int) -> _vp:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return _vp(stream.cuda_stream)


# ---------------------------------------------------------------- raw C-ABI mirrors
def stap_abi_version() -> int:
    return int(_lib.stap_abi_version())


def stap_status_string(code: int) -> str:
    return _lib.stap_status_string(code).decode()


def stap_plan_create(params: stap_params) -> int:
    h = _vp()
    _check(_lib.stap_plan_create(ctypes.byref(params), ctypes.byref(h)), "stap_plan_create")
    return h.value


def stap_plan_destroy(plan: int) -> None:
    _check(_lib.stap_plan_destroy(_vp(plan)), "stap_plan_destroy")


def stap_plan_workspace_bytes(plan: int, host_io: bool = False) -> int:
    n = ctypes.c_size_t()
    _check(_lib.stap_plan_workspace_bytes(_vp(plan), int(host_io), ctypes.byref(n)), "stap_plan_workspace_bytes")
    return int(n.value)


def stap_plan_describe(plan: int) -> str:
    return _lib.stap_plan_describe(_vp(plan)).decode()


def stap_doppler(plan: int, window, raw, cube, stream) -> None:
    _check(_lib.stap_doppler(_vp(plan), _ptr(window), _ptr(raw), _ptr(cube), stream), "stap_doppler")


def stap_covariance(plan: int, cube, cov, stream) -> None:
    _check(_lib.stap_covariance(_vp(plan), _ptr(cube), _ptr(cov), stream), "stap_covariance")


def stap_solve_weights(plan: int, cov, steering, weights, gamma, info, stream) -> None:
    _check(_lib.stap_solve_weights(_vp(plan), _ptr(cov), _ptr(steering), _ptr(weights), _ptr(gamma),
                                   _ptr(info), stream), "stap_solve_weights")


def stap_apply(plan: int, cube, weights, out, stream) -> None:
    _check(_lib.stap_apply(_vp(plan), _ptr(cube), _ptr(weights), _ptr(out), stream), "stap_apply")


def stap_run(plan: int, cube, steering, out, info, workspace, workspace_bytes: int, stream) -> None:
    _check(_lib.stap_run(_vp(plan), _ptr(cube), _ptr(steering), _ptr(out), _ptr(info), _ptr(workspace),
                         workspace_bytes, stream), "stap_run")


def stap_run_host(plan: int, h_cube, h_steering, h_out, h_info, workspace, workspace_bytes: int, stream) -> None:
    _check(_lib.stap_run_host(_vp(plan), _ptr(h_cube), _ptr(h_steering), _ptr(h_out), _ptr(h_info),
                              _ptr(workspace), workspace_bytes, stream), "stap_run_host")


# ---------------------------------------------------------------- convenience wrapper
@dataclass
class Dims:
    """Dimensions in the paper's vocabulary (PAPER.md:604-605 + north_star)."""
    C: int
    T: int
    D: int
    R: int
    K: int
    S: int
    lam: float = 1e-2

    @property
    def N(self) -> int:
        return self.C * self.T

    @property
    def B(self) -> int:
        return self.R // self.K


class StapPlan:
    """Owns a libstap plan; methods take torch tensors on the plan's device."""

    def __init__(self, dims: Dims, dop_begin: int = 0, dop_count: int | None = None, cube_bin0: int = 0,
                 cube_bins: int | None = None, batch: int = 1, device: int = 0, path: str = "auto",
                 out_multicast: bool = False, out_peer_offsets=(), precision: str = "fp32"):
        self.dims = dims
        self.dop_begin = dop_begin
        self.dop_count = dims.D if dop_count is None else dop_count
        self.cube_bin0 = cube_bin0
        self.cube_bins = dims.D if cube_bins is None else cube_bins
        self.batch = batch
        self.device = device
        self.params = stap_params(dims.C, dims.T, dims.D, dims.R, dims.K, dims.S, float(dims.lam), dop_begin,
                                  self.dop_count, cube_bin0, self.cube_bins, batch, device,
                                  PATHS[path], int(bool(out_multicast)), len(out_peer_offsets),
                                  (ctypes.c_int64 * 7)(*out_peer_offsets), PRECISIONS[precision])
        self.precision = precision
        self.remote_out = bool(out_multicast) or len(out_peer_offsets) > 0
        self.handle = stap_plan_create(self.params)
        self.workspace_bytes = stap_plan_workspace_bytes(self.handle, False)
        self.host_workspace_bytes = stap_plan_workspace_bytes(self.handle, True)
        self.description = stap_plan_describe(self.handle)
        self._ws = None

    def __del__(self, _destroy=_lib.stap_plan_destroy, _vp=_vp):
        # the defaults keep the C function reachable during interpreter shutdown
        h = getattr(self, "handle", None)
        if h:
            _destroy(_vp(h))
            self.handle = None

    # shapes ------------------------------------------------------------
    @property
    def cube_shape(self):
        d = self.dims
        return (self.batch, self.cube_bins, d.C, d.R)

    @property
    def out_shape(self):
        d = self.dims
        return (self.batch, self.dop_count, d.S, d.R)

    @property
    def cov_shape(self):
        d = self.dims
        return (self.batch, self.dop_count, d.B, d.N, d.N)

    @property
    def weights_shape(self):
        d = self.dims
        return (self.batch, self.dop_count, d.B, d.S, d.N)

    @property
    def info_shape(self):
        return (self.batch, self.dop_count, self.dims.B)

    def _chk(self, t, shape, dtype, name):
        import torch
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{name} must be a torch tensor")
        if t.dtype != dtype or not t.is_contiguous() or t.device != torch.device("cuda", self.device):
            raise ValueError(f"{name}: need contiguous {dtype} on cuda:{self.device}, got {t.dtype} on {t.device}")
        if tuple(t.shape) != tuple(shape) and t.numel() != _numel(shape):
            raise ValueError(f"{name}: shape {tuple(t.shape)} != {tuple(shape)}")

    def _out(self, out, shape, dtype, name, dev):
        """A caller's output tensor is checked like an input; a fresh one is allocated when None.
        A raw int device address is accepted only for `out` of a plan whose stores are remote
        (out_multicast / out_peer_offsets): the caller owns its mapping and extent."""
        import torch
        if out is None:
            return torch.empty(shape, dtype=dtype, device=dev)
        if isinstance(out, int):
            if name != "out" or not self.remote_out:
                raise TypeError(f"{name}: a raw address is only accepted for `out` of a remote-store plan")
            return out
        self._chk(out, shape, dtype, name)
        return out

    # stages ------------------------------------------------------------
    def doppler(self, raw, window, cube=None, stream=None):
        """The datacube from raw pulses [batch][D][C][R] (stap_doppler): taper + FFT along pulses."""
        import torch
        self._chk(raw, self.cube_shape, torch.complex64, "raw")
        if window.dtype != torch.float32 or window.shape != (self.dims.D,) or window.device != raw.device:
            raise ValueError("window: float32 [D] on the cube's device")
        cube = self._out(cube, self.cube_shape, torch.complex64, "cube", raw.device)
        stap_doppler(self.handle, window.contiguous(), raw, cube, _stream(stream, self.device))
        return cube

    def covariance(self, cube, cov=None, stream=None):
        import torch
        self._chk(cube, self.cube_shape, torch.complex64, "cube")
        cov = self._out(cov, self.cov_shape, torch.complex64, "cov", cube.device)
        stap_covariance(self.handle, cube, cov, _stream(stream, self.device))
        return cov

    def solve_weights(self, cov, steering, weights=None, gamma=None, info=None, stream=None):
        import torch
        d = self.dims
        self._chk(cov, self.cov_shape, torch.complex64, "cov")
        self._chk(steering, (d.S, d.N), torch.complex64, "steering")
        dev = cov.device
        weights = self._out(weights, self.weights_shape, torch.complex64, "weights", dev)
        gamma = self._out(gamma, self.info_shape + (d.S,), torch.float32, "gamma", dev)
        info = self._out(info, self.info_shape, torch.int32, "info", dev)
        stap_solve_weights(self.handle, cov, steering, weights, gamma, info, _stream(stream, self.device))
        return weights, gamma, info

    def apply(self, cube, weights, out=None, stream=None):
        import torch
        self._chk(cube, self.cube_shape, torch.complex64, "cube")
        self._chk(weights, self.weights_shape, torch.complex64, "weights")
        out = self._out(out, self.out_shape, torch.complex64, "out", cube.device)
        stap_apply(self.handle, cube, weights, out, _stream(stream, self.device))
        return out

    def workspace(self):
        import torch
        if self._ws is None or self._ws.numel() < max(self.workspace_bytes, 1):
            self._ws = torch.empty(max(self.workspace_bytes, 16), dtype=torch.uint8, device=f"cuda:{self.device}")
        return self._ws

    def run(self, cube, steering, out=None, info=None, stream=None):
        import torch
        d = self.dims
        self._chk(cube, self.cube_shape, torch.complex64, "cube")
        self._chk(steering, (d.S, d.N), torch.complex64, "steering")
        dev = cube.device
        out = self._out(out, self.out_shape, torch.complex64, "out", dev)
        info = self._out(info, self.info_shape, torch.int32, "info", dev)
        ws = self.workspace()
        stap_run(self.handle, cube, steering, out, info, ws, self.workspace_bytes, _stream(stream, self.device))
        return out, info

    def run_host(self, h_cube, h_steering, h_out, h_info, workspace, stream=None):
        """Host buffers (pinned torch CPU tensors) in and out; caller synchronises `stream`."""
        import torch
        d = self.dims
        for t, shape, dt, name in ((h_cube, self.cube_shape, torch.complex64, "h_cube"),
                                   (h_steering, (d.S, d.N), torch.complex64, "h_steering"),
                                   (h_out, self.out_shape, torch.complex64, "h_out"),
                                   (h_info, self.info_shape, torch.int32, "h_info")):
            if not isinstance(t, torch.Tensor) or t.device.type != "cpu" or t.dtype != dt or not t.is_contiguous() \
                    or t.numel() != _numel(shape):
                raise ValueError(f"{name}: need a contiguous {dt} host tensor of shape {shape}")
        self._chk(workspace, (workspace.numel(),), torch.uint8, "workspace")
        if workspace.numel() < self.host_workspace_bytes:
            raise ValueError("workspace: smaller than stap_plan_workspace_bytes(plan, 1)")
        stap_run_host(self.handle, h_cube, h_steering, h_out, h_info, workspace, self.host_workspace_bytes,
                      _stream(stream, self.device))


class StapComm:
    """The multi-GPU extension (include/stap.h): an NCCL communicator over the ranks' shards.
    StapComm(devices=[0, 1]) drives several GPUs from one process; StapComm(nranks=, rank=,
    uid=, device=) is one process's rank (uid from StapComm.unique_id() on one rank)."""

    def __init__(self, devices=None, nranks=None, rank=None, uid=None, device=None):
        h = _vp()
        if devices is not None:
            arr = (ctypes.c_int32 * len(devices))(*devices)
            _check(_lib.stap_comm_create(len(devices), arr, ctypes.byref(h)), "stap_comm_create")
            self.devices = list(devices)
        else:
            _check(_lib.stap_comm_init_rank(nranks, rank, bytes(uid), device, ctypes.byref(h)), "stap_comm_init_rank")
            self.devices = [device]
        self.handle = h.value
        n, l = ctypes.c_int32(), ctypes.c_int32()
        _check(_lib.stap_comm_size(_vp(self.handle), ctypes.byref(n), ctypes.byref(l)), "stap_comm_size")
        self.nranks, self.nlocal = n.value, l.value

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(_lib.stap_comm_unique_id(buf), "stap_comm_unique_id")
        return buf.raw

    def __del__(self, _destroy=_lib.stap_comm_destroy, _vp=_vp):
        h = getattr(self, "handle", None)
        if h:
            _destroy(_vp(h))
            self.handle = None

    def allgather_out(self, out_full, plans, streams=None):
        """In-place all-gather: out_full[i] [nranks][batch][Dl][S][R] on local device i."""
        import torch
        n = self.nlocal
        if streams is None:
            streams = [torch.cuda.current_stream(d) for d in self.devices]
        bufs = (_vp * n)(*[_ptr(t) for t in out_full])
        pls = (_vp * n)(*[p.handle for p in plans])
        sts = (_vp * n)(*[s.cuda_stream for s in streams])
        _check(_lib.stap_comm_allgather_out(_vp(self.handle), bufs, pls, sts), "stap_comm_allgather_out")

    def push_out(self, out_full, plans, streams=None):
        """Copy-engine gather: this rank's slice of out_full[i] into every peer's out_full."""
        import torch
        n = self.nlocal
        if streams is None:
            streams = [torch.cuda.current_stream(d) for d in self.devices]
        bufs = (_vp * n)(*[_ptr(t) for t in out_full])
        pls = (_vp * n)(*[p.handle for p in plans])
        sts = (_vp * n)(*[s.cuda_stream for s in streams])
        _check(_lib.stap_comm_push_out(_vp(self.handle), bufs, pls, sts), "stap_comm_push_out")

    def peer_offsets(self, out_full):
        """Per local device, the byte offsets for stap_params.out_peer_offset (collective)."""
        n = self.nlocal
        bufs = (_vp * n)(*[_ptr(t) for t in out_full])
        offs = (ctypes.c_int64 * (7 * n))()
        npeers = ctypes.c_int32()
        _check(_lib.stap_comm_peer_offsets(_vp(self.handle), bufs, offs, ctypes.byref(npeers)),
               "stap_comm_peer_offsets")
        return [tuple(offs[7 * i:7 * i + npeers.value]) for i in range(n)]


def _numel(shape):
    n = 1
    for s in shape:
        n *= s
    return n

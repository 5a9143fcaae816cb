"""fp64 CPU oracle for the STAP hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product package ``paper_2203_06233_b200`` never imports it, and this package
never imports the product package: the two share no code.

The arithmetic lives in ``oracle/stap_oracle.c`` (plain C11, fp64, explicit
re/im, ascending-order sums); this module only compiles it with gcc and
marshals numpy arrays through ctypes.  See the C file's header for the
passages and DESIGN.md readings it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "stap_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc -O2, no fast-math, no FMA contraction, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        cmd = ["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _LIB)
    return _LIB


class _Params(ctypes.Structure):
    _fields_ = [
        ("n_chan", ctypes.c_int32), ("tdof", ctypes.c_int32), ("n_dop", ctypes.c_int32),
        ("n_range", ctypes.c_int32), ("training_block", ctypes.c_int32),
        ("n_steering", ctypes.c_int32), ("diag_load", ctypes.c_double),
        ("dop_begin", ctypes.c_int32), ("dop_count", ctypes.c_int32),
        ("cube_bin0", ctypes.c_int32), ("cube_bins", ctypes.c_int32),
    ]


@dataclass
class OracleParams:
    """Dimensions in the paper's vocabulary plus the
    DESIGN.md readings: C channels, T TDOF, D Doppler bins, R range cells,
    K training block, S steering vectors, lambda relative diagonal loading."""
    C: int
    T: int
    D: int
    R: int
    K: int
    S: int
    lam: float = 1e-2
    dop_begin: int = 0
    dop_count: int | None = None
    cube_bin0: int = 0
    cube_bins: int | None = None

    @property
    def N(self) -> int:
        return self.C * self.T

    @property
    def B(self) -> int:
        return self.R // self.K

    @property
    def Dloc(self) -> int:
        return self.D if self.dop_count is None else self.dop_count

    def _c(self) -> _Params:
        return _Params(self.C, self.T, self.D, self.R, self.K, self.S, float(self.lam),
                       self.dop_begin, self.Dloc, self.cube_bin0,
                       self.D if self.cube_bins is None else self.cube_bins)


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.POINTER(_Params)
            vp = ctypes.c_void_p
            lib.stap_oracle_covariance.argtypes = [P, vp, vp, vp]
            lib.stap_oracle_solve.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, vp, vp, vp, vp, vp]
            lib.stap_oracle_solve_f64.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, vp, vp, vp, vp, vp]
            lib.stap_oracle_cholesky_f64.argtypes = [ctypes.c_int32, vp, vp]
            lib.stap_oracle_apply.argtypes = [P, vp, vp, vp]
            lib.stap_oracle_doppler.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                vp, vp, vp, ctypes.c_int32]
            lib.stap_oracle_run.argtypes = [P, vp, vp, vp, vp, vp, vp, vp, ctypes.c_int32]
            lib.stap_oracle_gj_inverse.argtypes = [ctypes.c_int32, vp, vp]
            for f in ("stap_oracle_covariance", "stap_oracle_solve", "stap_oracle_solve_f64",
                      "stap_oracle_cholesky_f64", "stap_oracle_apply", "stap_oracle_run",
                      "stap_oracle_gj_inverse", "stap_oracle_max_threads", "stap_oracle_doppler"):
                getattr(lib, f).restype = ctypes.c_int
            _lib = lib
    return _lib


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


def _c64(a) -> np.ndarray:
    a = np.ascontiguousarray(a)
    if a.dtype != np.complex64:
        raise TypeError(f"oracle inputs are the complex64 bytes the GPU sees; got {a.dtype}")
    return a


def _check(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"{what}: oracle returned {rc}")


def max_threads() -> int:
    return int(_load().stap_oracle_max_threads())


def covariance(p: OracleParams, cube) -> tuple[np.ndarray, np.ndarray]:
    """Loaded covariance Rm = Rhat + delta I per owned unit: [Dloc][B][N][N] complex128, delta [Dloc][B]."""
    cube = _c64(cube)
    R = np.zeros((p.Dloc, p.B, p.N, p.N), np.complex128)
    delta = np.zeros((p.Dloc, p.B), np.float64)
    pc = p._c()
    _check(_load().stap_oracle_covariance(ctypes.byref(pc), _ptr(cube), _ptr(R), _ptr(delta)), "covariance")
    return R, delta


def solve(Rm, steering) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """MVDR weights for matrices Rm [..., N, N] (complex64 -> promoted, or complex128 as given)
    and steering [S][N]: returns W [..., S, N], gamma [..., S], info [...]."""
    Rm = np.ascontiguousarray(Rm)
    batch = Rm.shape[:-2]
    N = Rm.shape[-1]
    S = steering.shape[0]
    cnt = int(np.prod(batch)) if batch else 1
    W = np.zeros(batch + (S, N), np.complex128)
    g = np.zeros(batch + (S,), np.float64)
    info = np.zeros(batch, np.int32) if batch else np.zeros((), np.int32)
    lib = _load()
    if Rm.dtype == np.complex64:
        st = _c64(steering)
        rc = lib.stap_oracle_solve(N, S, cnt, _ptr(Rm), _ptr(st), _ptr(W), _ptr(g), _ptr(info))
    elif Rm.dtype == np.complex128:
        st = np.ascontiguousarray(steering, np.complex128)
        rc = lib.stap_oracle_solve_f64(N, S, cnt, _ptr(Rm), _ptr(st), _ptr(W), _ptr(g), _ptr(info))
    else:
        raise TypeError(Rm.dtype)
    _check(rc, "solve")
    return W, g, info


def cholesky(Rm) -> tuple[np.ndarray, int]:
    Rm = np.ascontiguousarray(Rm, np.complex128)
    N = Rm.shape[0]
    L = np.zeros((N, N), np.complex128)
    info = _load().stap_oracle_cholesky_f64(N, _ptr(Rm), _ptr(L))
    return L, int(info)


def apply(p: OracleParams, cube, W) -> np.ndarray:
    """Y [Dloc][S][R] from complex64 cube and complex64 weights [Dloc][B][S][N]."""
    cube = _c64(cube)
    W = _c64(W)
    Y = np.zeros((p.Dloc, p.S, p.R), np.complex128)
    pc = p._c()
    _check(_load().stap_oracle_apply(ctypes.byref(pc), _ptr(cube), _ptr(W), _ptr(Y)), "apply")
    return Y


def run(p: OracleParams, cube, steering, nthreads: int = 1, intermediates: bool = False) -> dict:
    """Whole path for one cube: Y [Dloc][S][R], info [Dloc][B]; optionally R, W, gamma."""
    cube = _c64(cube)
    st = _c64(steering)
    Y = np.zeros((p.Dloc, p.S, p.R), np.complex128)
    info = np.zeros((p.Dloc, p.B), np.int32)
    R = W = g = None
    if intermediates:
        R = np.zeros((p.Dloc, p.B, p.N, p.N), np.complex128)
        W = np.zeros((p.Dloc, p.B, p.S, p.N), np.complex128)
        g = np.zeros((p.Dloc, p.B, p.S), np.float64)
    pc = p._c()
    nul = ctypes.c_void_p(0)
    rc = _load().stap_oracle_run(ctypes.byref(pc), _ptr(cube), _ptr(st), _ptr(Y), _ptr(info),
                                 _ptr(R) if R is not None else nul, _ptr(W) if W is not None else nul,
                                 _ptr(g) if g is not None else nul, int(nthreads))
    _check(rc, "run")
    out = {"Y": Y, "info": info}
    if intermediates:
        out.update(R=R, W=W, gamma=g)
    return out


def gj_inverse(A) -> np.ndarray:
    A = np.ascontiguousarray(A, np.complex128)
    n = A.shape[0]
    Ainv = np.zeros_like(A)
    rc = _load().stap_oracle_gj_inverse(n, _ptr(A), _ptr(Ainv))
    if rc:
        raise np.linalg.LinAlgError("singular")
    return Ainv


def doppler(window, raw, nthreads: int = 1) -> np.ndarray:
    """Doppler front end: X[n][d][c][r] = sum_p w[p] x[n][p][c][r] exp(-2 pi i p d / D), from
    complex64 raw [batch][D][C][R] (a 3-D array is one cube) and float32 window [D]; complex128 out."""
    raw = _c64(raw)
    one = raw.ndim == 3
    if one:
        raw = raw[None]
    n, D, C, R = raw.shape
    w = np.ascontiguousarray(window, np.float32)
    if w.shape != (D,):
        raise ValueError("window must have D entries")
    out = np.zeros(raw.shape, np.complex128)
    _check(_load().stap_oracle_doppler(D, C, R, n, _ptr(w), _ptr(raw), _ptr(out), int(nthreads)), "doppler")
    return out[0] if one else out

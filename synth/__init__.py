"""Seeded synthetic STAP inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the STAP method (no covariance, loading,
factorisation, solve or weighting).  It only fixes the workload shapes
(BASELINE.json ``configs``) and draws reproducible radar-like datacubes and
steering vectors with a counter-based generator, so that the oracle and every
GPU shard can be fed the exact same complex64 bytes.

Recipe:
  * splitmix64 counter generator: key_q = splitmix64(seed) ^ (q * 0xD1B54A32D192ED03);
    sample n of stream q uses u1 = splitmix64(key_q + 2n), u2 = splitmix64(key_q + 2n + 1);
    U1 = ((u1 >> 11) + 1) 2^-53 in (0, 1], U2 = (u2 >> 11) 2^-53;
    CN(0,1) = sqrt(-ln U1) (cos 2 pi U2 + i sin 2 pi U2), all in fp64.
  * datacube X[a][c][r] (Doppler bin a, channel c, range cell r -- the paper's
    "pulses x channels x samples per pulse", after the
    per-row Doppler FFT):
        noise CN(0,1)                                 stream 0, index (a*C + c)*R + r
      + sqrt(CNR) g_cl(a,r) exp(i pi c u_cl(a))       stream 1, index a*R + r, u_cl(a) = 2a/D - 1
      + sum_j sqrt(INR) g_j(a,r) exp(i pi c u_j)      streams 2,3; u = -0.35, +0.6
      + 8 point targets, |alpha| = sqrt(10)           stream 4
    CNR = INR = 30 dB.  Summed in fp64, rounded once to complex64.
  * steering: "ula" s_k[t*C + c] = exp(i pi c u_k) at t = h, else 0,
    u_k = -0.75 + 1.5 k / (S - 1); or "random" CN(0,1) stream 5, index k*N + i.
  * closed-form cubes E1 (DFT-white), E2 (geometric rank one) used by the pins.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)
_STREAM = 0xD1B54A32D192ED03


@dataclass(frozen=True)
class StapConfig:
    """One BASELINE.json workload.  C channels, T TDOF, D Doppler bins, R range
    cells, S steering vectors, K training block (R % K == 0), lam relative
    diagonal loading (reading c-6), cfg_id for the seeds."""
    name: str
    C: int
    T: int
    D: int
    R: int
    S: int
    K: int
    lam: float = 1e-2
    cfg_id: int = 0

    @property
    def N(self) -> int:
        return self.C * self.T

    @property
    def B(self) -> int:
        return self.R // self.K

    @property
    def h(self) -> int:
        return (self.T - 1) // 2

    def with_(self, **kw) -> "StapConfig":
        return replace(self, **kw)


# BASELINE.json configs[0..4].  K for tiny/medium/large is DESIGN.md reading c-8
# (smallest power of two >= 2N dividing R); small's K = 32 is given by BASELINE.json.
CONFIGS = {
    "tiny": StapConfig("tiny", C=2, T=2, D=8, R=64, S=4, K=16, cfg_id=1),
    "small": StapConfig("small", C=4, T=3, D=256, R=512, S=16, K=32, cfg_id=2),
    "medium": StapConfig("medium", C=6, T=5, D=512, R=1024, S=16, K=64, cfg_id=3),
    "large": StapConfig("large", C=8, T=7, D=1024, R=4096, S=16, K=128, cfg_id=4),
}


def weak_config(n_gpus: int) -> StapConfig:
    """BASELINE.json configs[4]: large shape with D = 1024 * G (fixed 1024-bin slice per GPU)."""
    return CONFIGS["large"].with_(name=f"weak{n_gpus}", D=1024 * n_gpus, cfg_id=5)


def splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (np.asarray(x, np.uint64) + _GOLD) & _M64
        z = ((z ^ (z >> np.uint64(30))) * _MIX1) & _M64
        z = ((z ^ (z >> np.uint64(27))) * _MIX2) & _M64
        return z ^ (z >> np.uint64(31))


def _key(seed: int, q: int) -> np.uint64:
    k = int(splitmix64(np.array([seed], np.uint64))[0])
    return np.uint64(k ^ ((q * _STREAM) & 0xFFFFFFFFFFFFFFFF))


def uniform_pair(seed: int, q: int, idx: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    key = _key(seed, q)
    idx = np.asarray(idx, np.uint64)
    with np.errstate(over="ignore"):
        u1 = splitmix64(key + np.uint64(2) * idx)
        u2 = splitmix64(key + np.uint64(2) * idx + np.uint64(1))
    U1 = ((u1 >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53
    U2 = (u2 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return U1, U2


def cn(seed: int, q: int, idx: np.ndarray) -> np.ndarray:
    """CN(0,1) samples of stream q at counter indices idx (complex128)."""
    U1, U2 = uniform_pair(seed, q, idx)
    mag = np.sqrt(-np.log(U1))
    ang = 2.0 * np.pi * U2
    return mag * (np.cos(ang) + 1j * np.sin(ang))


def cube_seed(cfg: StapConfig, cube_idx: int) -> int:
    return 1000 * cfg.cfg_id + cube_idx


def steering_seed(cfg: StapConfig) -> int:
    return 9000 + cfg.cfg_id


def _targets(cfg: StapConfig, seed: int, n_targets: int = 8):
    key = _key(seed, 4)
    m = np.arange(n_targets, dtype=np.uint64)
    with np.errstate(over="ignore"):
        v = [splitmix64(key + np.uint64(4) * m + np.uint64(o)) for o in range(4)]
    a = (v[0] % np.uint64(cfg.D)).astype(np.int64)
    r = (v[1] % np.uint64(cfg.R)).astype(np.int64)
    k = (v[2] % np.uint64(cfg.S)).astype(np.int64)
    phi = 2.0 * np.pi * (v[3] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return a, r, k, phi


def _ula_u(cfg: StapConfig) -> np.ndarray:
    if cfg.S == 1:
        return np.zeros(1)
    return -0.75 + 1.5 * np.arange(cfg.S) / (cfg.S - 1)


def datacube_bins(cfg: StapConfig, bins: np.ndarray, cube_idx: int = 0,
                  cnr_db: float = 30.0, inr_db: float = 30.0, n_targets: int = 8) -> np.ndarray:
    """Radar-like cube rows for the given global Doppler bins (any order, wrapping
    handled by the caller): complex64 [len(bins)][C][R]."""
    seed = cube_seed(cfg, cube_idx)
    bins = np.asarray(bins, np.int64) % cfg.D
    C, R, D = cfg.C, cfg.R, cfg.D
    a = bins[:, None, None]
    c = np.arange(C)[None, :, None]
    r = np.arange(R)[None, None, :]
    x = cn(seed, 0, (a * C + c) * R + r)
    ar = (bins[:, None] * R + np.arange(R)[None, :])[:, None, :]
    sc = np.sqrt(10.0 ** (cnr_db / 10.0))
    si = np.sqrt(10.0 ** (inr_db / 10.0))
    u_cl = (2.0 * bins / D - 1.0)[:, None, None]
    x = x + sc * cn(seed, 1, ar) * np.exp(1j * np.pi * c * u_cl)
    for q, u in ((2, -0.35), (3, 0.6)):
        x = x + si * cn(seed, q, ar) * np.exp(1j * np.pi * c * u)
    ta, tr, tk, tphi = _targets(cfg, seed, n_targets)
    uk = _ula_u(cfg)
    pos = {int(b): i for i, b in enumerate(bins)}
    for m in range(n_targets):
        i = pos.get(int(ta[m]))
        if i is None:
            continue
        alpha = np.sqrt(10.0) * np.exp(1j * tphi[m])
        x[i, :, tr[m]] += alpha * np.exp(1j * np.pi * np.arange(C) * uk[tk[m]])
    return x.astype(np.complex64)


def datacube(cfg: StapConfig, cube_idx: int = 0, **kw) -> np.ndarray:
    """Full cube [D][C][R] complex64."""
    return datacube_bins(cfg, np.arange(cfg.D), cube_idx, **kw)


def shard_window(cfg: StapConfig, dop_begin: int, dop_count: int) -> tuple[int, int]:
    """(cube_bin0, cube_bins) of the smallest cube buffer that serves the owned
    bins [dop_begin, dop_begin + dop_count): the slice plus T-1 halo bins, or the
    whole cube when that is no larger.  Window placement = DESIGN.md reading c-2."""
    nb = dop_count + cfg.T - 1
    if nb >= cfg.D:
        return 0, cfg.D
    return (dop_begin - cfg.h) % cfg.D, nb


def shard_range(D: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous chunk rule: rank g owns [g*ceil(D/G), min(D, (g+1)*ceil(D/G)))."""
    chunk = -(-D // world)
    lo = min(D, rank * chunk)
    hi = min(D, lo + chunk)
    return lo, hi - lo


def steering(cfg: StapConfig, kind: str = "ula") -> np.ndarray:
    """Steering vectors [S][N] complex64, element i = t*C + c (reading c-4)."""
    S, N, C = cfg.S, cfg.N, cfg.C
    if kind == "ula":
        s = np.zeros((S, cfg.T, C), np.complex128)
        s[:, cfg.h, :] = np.exp(1j * np.pi * np.arange(C)[None, :] * _ula_u(cfg)[:, None])
        return s.reshape(S, N).astype(np.complex64)
    if kind == "random":
        idx = np.arange(S * N).reshape(S, N)
        return cn(steering_seed(cfg), 5, idx).astype(np.complex64)
    raise ValueError(kind)


def cube_e1(cfg: StapConfig) -> np.ndarray:
    """DFT-white cube (pin E1): X[a][c][r] = exp(2 pi i (a C + c)(r mod K) / K).
    Every window then has Rhat = I exactly when N <= K and K | D*C."""
    a = np.arange(cfg.D)[:, None, None]
    c = np.arange(cfg.C)[None, :, None]
    r = np.arange(cfg.R)[None, None, :]
    ph = ((a * cfg.C + c) * (r % cfg.K)) % cfg.K
    return np.exp(2j * np.pi * ph / cfg.K).astype(np.complex64)


def cube_e2(cfg: StapConfig, seed: int = 77):
    """Geometric rank-one cube (pin E2): X[a][c][r] = c_r g_c rho^a with rho = i
    (m = D/4, so D % 4 == 0), g_c = i^(c mod 4) and Gaussian-integer c_r drawn from
    stream 6.  Every product is a small Gaussian integer, so the complex64 cube
    is exactly rank one in every window.  Returns (cube complex64, c_r, g, rho)."""
    if cfg.D % 4:
        raise ValueError("cube_e2 needs D % 4 == 0 (rho = i)")
    U1, U2 = uniform_pair(seed, 6, np.arange(cfg.R))
    cr = (1.0 + np.floor(U1 * 3.0)) + 1j * (np.floor(U2 * 3.0) - 1.0)
    g = (1j) ** (np.arange(cfg.C) % 4)
    rho = 1j
    rho_a = (1j) ** (np.arange(cfg.D) % 4)
    x = rho_a[:, None, None] * g[None, :, None] * cr[None, None, :]
    return x.astype(np.complex64), cr, g, rho

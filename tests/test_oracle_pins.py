"""Pins for the fp64 oracle (-m "not gpu").

The oracle (oracle/stap_oracle.c) is checked against things other than
itself: hand-worked fixtures (tests/golden), closed forms (E1 DFT-white cube,
E2 rank-one cube via Sherman-Morrison, E3 target injection, identity
covariance), exact rational arithmetic on tiny integer inputs, library
special cases (numpy.linalg.inv / eigvalsh, an independent Gauss-Jordan),
the MVDR optimality conditions, and the invariances that the DESIGN.md
readings imply (phase, scale, channel permutation, Doppler roll, block and
bin locality).  Each test names the pin id of SURVEY.md 8(c) c.4 / DESIGN.md.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from oracle import OracleParams

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def P(cfg, **kw):
    return OracleParams(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam, **kw)


def relerr(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        g = json.load(f)
    p = g["params"]
    cube = (np.array(g["cube_re"]) + 1j * np.array(g["cube_im"])).astype(np.complex64)
    st = (np.array(g["steering_re"]) + 1j * np.array(g["steering_im"])).astype(np.complex64)
    op = OracleParams(p["C"], p["T"], p["D"], p["R"], p["K"], p["S"], p["lam"])
    return g, op, cube, st


# ---------------------------------------------------------------- golden fixtures
def test_golden_hand_n2():
    g, op, cube, st = _golden("hand_n2.json")
    out = oracle.run(op, cube, st, intermediates=True)
    Rm = np.array(g["Rm_re"]) + 1j * np.array(g["Rm_im"])
    W = np.array(g["W_re"]) + 1j * np.array(g["W_im"])
    Y = np.array(g["Y_re"]) + 1j * np.array(g["Y_im"])
    assert np.abs(out["R"][0, 0] - Rm).max() < 1e-15
    assert np.abs(out["W"][0, 0] - W).max() < 1e-15
    assert abs(out["gamma"][0, 0, 0] - g["gamma"][0]) < 1e-14
    assert np.abs(out["Y"][0] - Y).max() < 1e-15
    assert out["info"][0, 0] == 0


def test_golden_hand_n1_P13():
    g, op, cube, st = _golden("hand_n1.json")
    out = oracle.run(op, cube, st)
    Y = np.array(g["Y_re"]) + 1j * np.array(g["Y_im"])
    assert np.abs(out["Y"][0] - Y).max() < 1e-15


# ---------------------------------------------------------------- exact rationals
class GQ:
    """Gaussian rational re + i im with exact Fractions (brute-force pin)."""

    def __init__(self, re, im=0):
        self.re, self.im = Fraction(re), Fraction(im)

    def __add__(s, o):
        return GQ(s.re + o.re, s.im + o.im)

    def __sub__(s, o):
        return GQ(s.re - o.re, s.im - o.im)

    def __mul__(s, o):
        return GQ(s.re * o.re - s.im * o.im, s.re * o.im + s.im * o.re)

    def conj(s):
        return GQ(s.re, -s.im)

    def __truediv__(s, o):
        den = o.re * o.re + o.im * o.im
        n = s * o.conj()
        return GQ(n.re / den, n.im / den)

    def c(self):
        return complex(float(self.re), float(self.im))


def _exact_mvdr(Z, s, lam):
    """Exact Y for one unit by Gaussian elimination (not Cholesky) in Q(i)."""
    N, K = len(Z), len(Z[0])
    R = [[GQ(0) for _ in range(N)] for _ in range(N)]
    for i in range(N):
        for l in range(N):
            acc = GQ(0)
            for j in range(K):
                acc = acc + Z[i][j] * Z[l][j].conj()
            R[i][l] = acc / GQ(K)
    tr = GQ(0)
    for i in range(N):
        tr = tr + R[i][i]
    delta = GQ(lam) * tr / GQ(N)
    for i in range(N):
        R[i][i] = R[i][i] + delta
    M = [row[:] + [s[i]] for i, row in enumerate(R)]
    for col in range(N):
        piv = next(r for r in range(col, N) if M[r][col].re != 0 or M[r][col].im != 0)
        M[col], M[piv] = M[piv], M[col]
        for r in range(N):
            if r != col:
                f = M[r][col] / M[col][col]
                M[r] = [a - f * b for a, b in zip(M[r], M[col])]
    v = [M[i][N] / M[i][i] for i in range(N)]
    gamma = GQ(0)
    for i in range(N):
        gamma = gamma + s[i].conj() * v[i]
    w = [vi / gamma for vi in v]
    Y = []
    for j in range(K):
        acc = GQ(0)
        for i in range(N):
            acc = acc + w[i].conj() * Z[i][j]
        Y.append(acc)
    return w, gamma, Y


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_exact_rational_brute_force(seed):
    """Tiny integer cube (C=2, T=2, D=3, K=6): exact Q(i) solve by Gauss elimination
    vs the oracle's fp64 Cholesky path.  Pins steps 1-6 incl. window + wrap."""
    rng = np.random.default_rng(seed)
    C, T, D, R, K, S = 2, 2, 3, 12, 6, 2
    lam = Fraction(1, 8)
    cube = (rng.integers(-3, 4, (D, C, R)) + 1j * rng.integers(-3, 4, (D, C, R))).astype(np.complex64)
    st = (rng.integers(-2, 3, (S, C * T)) + 1j * rng.integers(-2, 3, (S, C * T))).astype(np.complex64)
    st[:, 0] += 3  # keep every steering vector nonzero
    op = OracleParams(C, T, D, R, K, S, float(lam))
    out = oracle.run(op, cube, st, intermediates=True)
    h = (T - 1) // 2
    for d in range(D):
        for b in range(R // K):
            Z = [[GQ(int(cube[(d - h + t) % D, c, b * K + j].real), int(cube[(d - h + t) % D, c, b * K + j].imag))
                  for j in range(K)] for t in range(T) for c in range(C)]
            for k in range(S):
                s = [GQ(int(x.real), int(x.imag)) for x in st[k]]
                w, gamma, Y = _exact_mvdr(Z, s, lam)
                assert np.abs(out["W"][d, b, k] - np.array([x.c() for x in w])).max() < 1e-13
                assert abs(out["gamma"][d, b, k] - gamma.c().real) < 1e-12 * abs(gamma.c())
                assert np.abs(out["Y"][d, k, b * K:(b + 1) * K] - np.array([y.c() for y in Y])).max() < 1e-12


# ---------------------------------------------------------------- closed forms
def test_E1_dft_white_exact_tiny():
    """E1 with K = 4 (exp(2 pi i m / 4) is exact in complex64): Rhat = I exactly,
    so Rm = (1 + lambda) I, w_k = s_k / ||s_k||^2, Y = s_k^H z / ||s_k||^2."""
    cfg = synth.CONFIGS["tiny"].with_(K=4)
    cube = synth.cube_e1(cfg)
    st = synth.steering(cfg, "random")
    out = oracle.run(P(cfg), cube, st, intermediates=True)
    eye = (1 + cfg.lam) * np.eye(cfg.N)
    assert np.abs(out["R"] - eye).max() < 1e-15
    s = st.astype(np.complex128)
    wexp = s / np.sum(np.abs(s) ** 2, axis=1, keepdims=True)
    assert np.abs(out["W"] - wexp[None, None]).max() < 1e-15
    h = cfg.h
    for d in range(cfg.D):
        Z = np.concatenate([cube[(d - h + t) % cfg.D] for t in range(cfg.T)], axis=0).astype(np.complex128)
        Yexp = wexp.conj() @ Z
        assert relerr(out["Y"][d], Yexp) < 1e-14


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_E1_dft_white_configs(name):
    """E1 at the config's own K: Rhat = I up to the complex64 rounding of X (~1e-7)."""
    cfg = synth.CONFIGS[name]
    cube = synth.cube_e1(cfg)
    st = synth.steering(cfg, "ula")
    out = oracle.run(P(cfg), cube, st, intermediates=True)
    assert np.abs(out["R"] - (1 + cfg.lam) * np.eye(cfg.N)).max() < 2e-6
    s = st.astype(np.complex128)
    wexp = s / np.sum(np.abs(s) ** 2, axis=1, keepdims=True)
    for d in (0, 1, cfg.D // 2, cfg.D - 1):
        Z = np.concatenate([cube[(d - cfg.h + t) % cfg.D] for t in range(cfg.T)], axis=0).astype(np.complex128)
        assert relerr(out["Y"][d], wexp.conj() @ Z) < 1e-5


@pytest.mark.parametrize("name,lam", [("tiny", 1e-2), ("tiny", 1e-3), ("small", 1e-2)])
def test_E2_rank_one_sherman_morrison(name, lam):
    """E2: X = c_r g_c rho^a (exact Gaussian integers) => Rhat = p_b a a^H,
    delta = lam p_b ||a||^2 / N, and by Sherman-Morrison (P10)
    v = (s - a (a^H s) p / (delta + p a^H a)) / delta; w = v / (s^H v);
    Y[d][k][r] = rho^(d-h) c_r (w^H a)."""
    cfg = synth.CONFIGS[name].with_(lam=lam)
    cube, cr, g, rho = synth.cube_e2(cfg)
    st = synth.steering(cfg, "random").astype(np.complex128)
    out = oracle.run(P(cfg), cube, st.astype(np.complex64), intermediates=True)
    a = np.concatenate([g * rho ** t for t in range(cfg.T)])
    N, K = cfg.N, cfg.K
    for b in range(cfg.B):
        pb = np.sum(np.abs(cr[b * K:(b + 1) * K]) ** 2) / K
        delta = lam * pb * np.vdot(a, a).real / N
        for d in (0, 1, cfg.D - 1):
            ph = rho ** ((d - cfg.h) % cfg.D)
            Rexp = pb * np.outer(a, a.conj()) + delta * np.eye(N)
            assert np.abs(out["R"][d, b] - Rexp).max() < 1e-13 * np.abs(Rexp).max()
            for k in range(cfg.S):
                s = st[k]
                v = (s - a * np.vdot(a, s) * pb / (delta + pb * np.vdot(a, a).real)) / delta
                w = v / np.vdot(s, v)
                assert relerr(out["W"][d, b, k], w) < 1e-12
                Yexp = ph * cr[b * K:(b + 1) * K] * np.vdot(w, a)
                scale = np.linalg.norm(w) * np.linalg.norm(a) * np.abs(cr[b * K:(b + 1) * K]).max()
                assert np.abs(out["Y"][d, k, b * K:(b + 1) * K] - Yexp).max() < 1e-12 * scale


def test_E3_target_injection():
    """E3 / P11: set the window bins of one (d, r) to alpha s_k: Y[d][k][r] = alpha (w^H s = 1).
    alpha and s are small Gaussian integers so alpha s_k is exact in complex64."""
    cfg = synth.CONFIGS["tiny"]
    cube = synth.datacube(cfg)
    rng = np.random.default_rng(3)
    st = (rng.integers(-3, 4, (cfg.S, cfg.N)) + 1j * rng.integers(-3, 4, (cfg.S, cfg.N))).astype(np.complex64)
    st[:, 0] += 4
    alpha = 3 - 2j
    for d, r, k in [(0, 5, 1), (3, 17, 0), (cfg.D - 1, 63, 3)]:
        x = cube.copy()
        for t in range(cfg.T):
            x[(d - cfg.h + t) % cfg.D, :, r] = alpha * st[k, t * cfg.C:(t + 1) * cfg.C]
        out = oracle.run(P(cfg), x, st)
        assert abs(out["Y"][d, k, r] - alpha) < 1e-12 * abs(alpha)


def test_P5_identity_covariance():
    """P5: R = I gives w_k = s_k / ||s_k||^2 and gamma_k = ||s_k||^2."""
    cfg = synth.CONFIGS["small"]
    st = synth.steering(cfg, "random").astype(np.complex128)
    R = np.broadcast_to(np.eye(cfg.N, dtype=np.complex128), (3, cfg.N, cfg.N)).copy()
    W, g, info = oracle.solve(R, st)
    n2 = np.sum(np.abs(st) ** 2, axis=1)
    assert np.all(info == 0)
    assert np.abs(g - n2[None]).max() < 1e-13 * n2.max()
    assert np.abs(W - (st / n2[:, None])[None]).max() < 1e-15


# ---------------------------------------------------------------- invariants / library special cases
@pytest.fixture(scope="module")
def small_run():
    cfg = synth.CONFIGS["small"].with_(D=16)
    cube = synth.datacube(cfg)
    st = synth.steering(cfg, "random")
    out = oracle.run(P(cfg), cube, st, intermediates=True, nthreads=4)
    return cfg, cube, st, out


def test_P2_P3_hermitian_and_trace(small_run):
    cfg, cube, st, out = small_run
    R = out["R"]
    assert np.array_equal(R, np.conj(np.swapaxes(R, -1, -2)))  # bitwise mirror
    assert np.all(np.diagonal(R, axis1=-2, axis2=-1).imag == 0)
    for d in (0, 7, 15):
        for b in (0, cfg.B - 1):
            Z = np.concatenate([cube[(d - cfg.h + t) % cfg.D, :, b * cfg.K:(b + 1) * cfg.K]
                                for t in range(cfg.T)], axis=0).astype(np.complex128)
            tr_exp = (1 + cfg.lam) * np.sum(np.abs(Z) ** 2) / cfg.K
            assert abs(np.trace(R[d, b]).real - tr_exp) < 1e-13 * tr_exp


def test_P4_psd(small_run):
    """Rhat is PSD: eig(Rm) >= delta; Cholesky of Rm - 0.99 delta I succeeds."""
    cfg, cube, st, out = small_run
    Rm = out["R"][:4].reshape(-1, cfg.N, cfg.N)
    for M in Rm:
        delta = cfg.lam * np.trace(M).real / (1 + cfg.lam) / cfg.N
        ev = np.linalg.eigvalsh(M)
        assert ev.min() >= delta * (1 - 1e-9)
        _, info = oracle.cholesky(M - 0.99 * delta * np.eye(cfg.N))
        assert info == 0
        L, info = oracle.cholesky(M)
        assert info == 0 and np.abs(L @ L.conj().T - M).max() < 1e-12 * np.abs(M).max()


def test_P6_P7_P8_P9_solve_identities(small_run):
    """P6 w^H s = 1; P7 (w^H Rm w) gamma = 1; P8 ||Rm v - s|| / ||s|| < 1e-10 with v = gamma w;
    P9 v agrees with numpy.linalg.inv and with the independent Gauss-Jordan inverse."""
    cfg, cube, st, out = small_run
    s = st.astype(np.complex128)
    for d in (0, 5, 15):
        for b in (0, 3, cfg.B - 1):
            M, W, g = out["R"][d, b], out["W"][d, b], out["gamma"][d, b]
            Minv_np = np.linalg.inv(M)
            Minv_gj = oracle.gj_inverse(M)
            kappa = np.linalg.cond(M)
            assert np.abs(Minv_gj @ M - np.eye(cfg.N)).max() < 1e-12 * kappa
            for k in range(cfg.S):
                w = W[k]
                assert abs(np.vdot(w, s[k]) - 1) < 1e-12
                assert abs(np.vdot(w, M @ w).real * g[k] - 1) < 1e-12
                v = g[k] * w
                assert np.linalg.norm(M @ v - s[k]) / np.linalg.norm(s[k]) < 1e-10
                assert relerr(v, Minv_np @ s[k]) < 1e-12 * kappa
                assert relerr(v, Minv_gj @ s[k]) < 1e-12 * kappa
                assert abs(g[k] - np.vdot(s[k], Minv_np @ s[k]).real) < 1e-12 * kappa * g[k]


def test_mvdr_optimality_brute_force(small_run):
    """w minimises w^H Rm w over {w : w^H s = 1}: random feasible perturbations never do better."""
    cfg, cube, st, out = small_run
    rng = np.random.default_rng(5)
    s = st.astype(np.complex128)
    M, W = out["R"][3, 2], out["W"][3, 2]
    for k in range(cfg.S):
        w = W[k]
        f0 = np.vdot(w, M @ w).real
        for _ in range(20):
            e = rng.standard_normal(cfg.N) + 1j * rng.standard_normal(cfg.N)
            e -= s[k] * np.vdot(s[k], e) / np.vdot(s[k], s[k])  # keep (w+e)^H s = 1
            e *= 1e-3 * np.linalg.norm(w) / np.linalg.norm(e)
            assert np.vdot(w + e, M @ (w + e)).real >= f0 * (1 - 1e-12)


def test_threads_bitwise(small_run):
    cfg, cube, st, out = small_run
    one = oracle.run(P(cfg), cube, st, nthreads=1)
    assert np.array_equal(one["Y"], out["Y"])


def test_staged_equals_run(small_run):
    """covariance -> solve -> apply on fp64 intermediates reproduces run (same sums, same order)."""
    cfg, cube, st, out = small_run
    R, delta = oracle.covariance(P(cfg), cube)
    assert np.array_equal(R, out["R"])
    assert np.allclose(delta, cfg.lam * np.trace(R, axis1=-2, axis2=-1).real / (1 + cfg.lam) / cfg.N, rtol=1e-13)
    W, g, info = oracle.solve(R, st.astype(np.complex128))
    assert np.array_equal(W, out["W"]) and np.all(info == 0)


# ---------------------------------------------------------------- invariances (P12)
def _y(cfg, cube, st, **kw):
    return oracle.run(P(cfg, **kw), cube, st)["Y"]


@pytest.fixture(scope="module")
def tiny():
    cfg = synth.CONFIGS["tiny"]
    return cfg, synth.datacube(cfg), synth.steering(cfg, "random")


def test_P12a_phase(tiny):
    cfg, cube, st = tiny
    Y0 = _y(cfg, cube, st)
    Y1 = _y(cfg, (1j * cube.astype(np.complex128)).astype(np.complex64), st)
    assert np.abs(Y1 - 1j * Y0).max() < 1e-14 * np.abs(Y0).max()


def test_P12b_scale(tiny):
    cfg, cube, st = tiny
    out0 = oracle.run(P(cfg), cube, st, intermediates=True)
    out1 = oracle.run(P(cfg), (cube * np.float32(2)).astype(np.complex64), st, intermediates=True)
    assert np.abs(out1["W"] - out0["W"]).max() < 1e-15 * np.abs(out0["W"]).max()
    assert np.abs(out1["Y"] - 2 * out0["Y"]).max() < 1e-14 * np.abs(out0["Y"]).max()


def test_P12c_channel_permutation(tiny):
    cfg, cube, st = tiny
    perm = np.array([1, 0])
    st_p = st.reshape(cfg.S, cfg.T, cfg.C)[:, :, perm].reshape(cfg.S, cfg.N)
    Y0 = _y(cfg, cube, st)
    Y1 = _y(cfg, np.ascontiguousarray(cube[:, perm, :]), np.ascontiguousarray(st_p))
    assert np.abs(Y1 - Y0).max() < 1e-12 * np.abs(Y0).max()


def test_P12d_doppler_roll(tiny):
    cfg, cube, st = tiny
    Y0 = _y(cfg, cube, st)
    for shift in (1, 3):
        Y1 = _y(cfg, np.ascontiguousarray(np.roll(cube, shift, axis=0)), st)
        assert np.array_equal(Y1, np.roll(Y0, shift, axis=0))


def test_P12e_block_locality(tiny):
    cfg, cube, st = tiny
    Y0 = _y(cfg, cube, st)
    x = cube.copy()
    x[:, :, 2 * cfg.K + 3] += 5 - 1j
    Y1 = _y(cfg, x, st)
    blk = np.zeros(cfg.R, bool)
    blk[2 * cfg.K:3 * cfg.K] = True
    assert np.array_equal(Y1[:, :, ~blk], Y0[:, :, ~blk])
    assert np.abs(Y1[:, :, blk] - Y0[:, :, blk]).max() > 1e-6


@pytest.mark.parametrize("T,a", [(2, 5), (3, 0), (3, 7)])
def test_P12f_window_and_wrap(T, a):
    """Perturbing bin a changes exactly the bins d with a in {d-h .. d-h+T-1} (mod D): readings c-2, c-3."""
    cfg = synth.CONFIGS["tiny"].with_(T=T)
    cube = synth.datacube(cfg)
    st = synth.steering(cfg, "random")
    Y0 = _y(cfg, cube, st)
    x = cube.copy()
    x[a] += 3 + 2j
    Y1 = _y(cfg, x, st)
    changed = {d for d in range(cfg.D) if not np.array_equal(Y1[d], Y0[d])}
    expect = {(a + cfg.h - t) % cfg.D for t in range(T)}
    assert changed == expect


# ---------------------------------------------------------------- degenerate cases / info (c-11)
def test_P14_zero_block_info():
    cfg = synth.CONFIGS["tiny"]
    cube = synth.datacube(cfg)
    st = synth.steering(cfg, "random")
    x = cube.copy()
    x[:, :, cfg.K:2 * cfg.K] = 0  # block 1 zero in every bin
    out = oracle.run(P(cfg), x, st, intermediates=True)
    assert np.all(out["info"][:, 1] == 1)
    assert np.all(out["W"][:, 1] == 0) and np.all(out["Y"][:, :, cfg.K:2 * cfg.K] == 0)
    assert np.all(out["info"][:, 0] == 0)


def test_zero_steering_info():
    cfg = synth.CONFIGS["tiny"]
    cube = synth.datacube(cfg)
    st = synth.steering(cfg, "random")
    st[2] = 0
    out = oracle.run(P(cfg), cube, st, intermediates=True)
    assert np.all(out["info"] == -3)
    assert np.all(out["Y"][:, 2] == 0) and np.all(out["W"][:, :, 2] == 0)
    assert np.all(out["Y"][:, 1] != 0)


def test_rank_one_zero_loading_info():
    """Exactly rank-one Rhat (all-ones cube, exact in fp64) with lambda = 0: pivot 2
    is exactly 0, so info = 2 and W = Y = 0 (reading c-11)."""
    cfg = synth.CONFIGS["tiny"].with_(lam=0.0)
    cube = np.ones((cfg.D, cfg.C, cfg.R), np.complex64)
    st = synth.steering(cfg, "random")
    out = oracle.run(P(cfg), cube, st, intermediates=True)
    assert np.all(out["info"] == 2)
    assert np.all(out["Y"] == 0) and np.all(out["W"] == 0)


# ---------------------------------------------------------------- shards (P15 on the oracle)
@pytest.mark.parametrize("G", [2, 3, 8])
def test_shard_windows_bitwise(G):
    """Doppler shards with slice+halo cube buffers reproduce the full-cube result bitwise."""
    cfg = synth.CONFIGS["tiny"].with_(T=3)
    cube = synth.datacube(cfg)
    st = synth.steering(cfg, "random")
    Yfull = _y(cfg, cube, st)
    parts = []
    for g in range(G):
        lo, cnt = synth.shard_range(cfg.D, G, g)
        if cnt == 0:
            continue
        b0, nb = synth.shard_window(cfg, lo, cnt)
        local = synth.datacube_bins(cfg, (b0 + np.arange(nb)) % cfg.D)
        parts.append(_y(cfg, local, st, dop_begin=lo, dop_count=cnt, cube_bin0=b0, cube_bins=nb))
    assert np.array_equal(np.concatenate(parts, axis=0), Yfull)


def test_generator_shard_consistency():
    cfg = synth.CONFIGS["small"]
    full = synth.datacube(cfg)
    bins = np.array([250, 255, 0, 1, 2])
    assert np.array_equal(synth.datacube_bins(cfg, bins), full[bins])


def test_generator_statistics():
    """CN(0,1): E|x|^2 = 1, E x = 0 (sanity of the input recipe, not of the method)."""
    x = synth.cn(123, 0, np.arange(200000))
    assert abs(np.mean(np.abs(x) ** 2) - 1) < 0.01
    assert abs(np.mean(x)) < 0.01


# ---------------------------------------------------------------- Doppler front end
def _raw(D, C, R, seed=0, n=None):
    rng = np.random.default_rng(seed)
    shape = (D, C, R) if n is None else (n, D, C, R)
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64)


def test_doppler_is_the_dft_numpy():
    """Special case reducing to a library routine: the windowed DFT along pulses = numpy.fft.fft."""
    D, C, R = 16, 3, 5
    x = _raw(D, C, R)
    w = np.hanning(D).astype(np.float32)
    X = oracle.doppler(w, x)
    ref = np.fft.fft(w.astype(np.float64)[:, None, None] * x.astype(np.complex128), axis=0)
    assert np.abs(X - ref).max() <= 1e-12 * np.abs(ref).max()


def test_doppler_parseval():
    D, C, R = 32, 2, 4
    x = _raw(D, C, R, seed=1)
    w = (0.5 + np.arange(D) / D).astype(np.float32)
    X = oracle.doppler(w, x)
    wx = w.astype(np.float64)[:, None, None] * x.astype(np.complex128)
    assert abs(np.sum(np.abs(X) ** 2) - D * np.sum(np.abs(wx) ** 2)) <= 1e-12 * D * np.sum(np.abs(wx) ** 2)


def test_doppler_tone_lands_in_its_bin():
    """x[p] = exp(+2 pi i f p / D), w = 1  ->  X[d] = D delta(d - f)  (sign convention of the transform)."""
    D, f = 64, 5
    p = np.arange(D)
    x = np.exp(2j * np.pi * f * p / D).astype(np.complex64)[:, None, None] * np.ones((1, 2, 3), np.complex64)
    X = oracle.doppler(np.ones(D, np.float32), x)
    expect = np.zeros(D)
    expect[f] = D
    assert np.abs(X[:, 1, 2] - expect).max() <= 1e-5 * D  # complex64 input rounding of the tone


def test_doppler_shift_theorem_and_batch():
    """A one-pulse circular delay multiplies bin d by exp(-2 pi i d / D); batched = per cube."""
    D, C, R = 16, 2, 3
    x = _raw(D, C, R, seed=2)
    w = np.ones(D, np.float32)
    X0 = oracle.doppler(w, x)
    X1 = oracle.doppler(w, np.roll(x, 1, axis=0))
    ramp = np.exp(-2j * np.pi * np.arange(D) / D)[:, None, None]
    assert np.abs(X1 - ramp * X0).max() <= 1e-12 * np.abs(X0).max()
    xb = _raw(D, C, R, seed=3, n=3)
    Xb = oracle.doppler(w, xb)
    for n in range(3):
        assert np.array_equal(Xb[n], oracle.doppler(w, xb[n]))

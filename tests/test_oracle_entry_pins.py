"""Pins for the oracle entry points the GPU parity tests use as checkers on their own
(-m "not gpu"): ``oracle.apply`` (given weights -> Y) and the complex64 ``oracle.solve``.

The whole-path ``oracle.run`` is pinned in test_oracle_pins.py; these two have their own
indexing (W32 [Dloc][B][S][N] and Y [Dloc][S][R] with shard offsets; the complex64
promotion) and are checked here against things other than themselves:

- apply: the hand-worked fixture tests/golden/hand_n2.json (its W, exactly representable
  in complex64, gives its Y), and an independent NumPy construction of the definition
  Y[d][k][r] = sum_i conj(W[d][b(r)][k][i]) z_{d,r}[i] (reading
  c-12), z built from the window rule of readings c-2/c-3/c-4, on tiny, small-shaped and
  sharded (dop_begin / cube_bin0 offset, wrapped) windows.
- solve (complex64 entry): bitwise equal to the fp64 entry on the exactly promoted
  matrices (so every pin of the fp64 path carries over), and the MVDR definition
  w = R^-1 s / (s^H R^-1 s) via numpy.linalg.solve (reading c-9).
"""
import json
import os

import numpy as np

import oracle
import synth
from oracle import OracleParams

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _window_Z(cube_local, cfg, d, b, bin0, nbins):
    """Independent snapshot matrix Z [N][K] of unit (d, b): z[t*C + c] = X[(d - h + t) mod D][c][r]."""
    rows = []
    for t in range(cfg.T):
        a = (d - cfg.h + t) % cfg.D
        rows.append(cube_local[(a - bin0) % cfg.D][:, b * cfg.K:(b + 1) * cfg.K])
    return np.concatenate(rows, 0).astype(np.complex128)


def _numpy_apply(cube_local, W, cfg, d0, cnt, bin0, nbins):
    Y = np.zeros((cnt, cfg.S, cfg.R), np.complex128)
    for dl in range(cnt):
        for b in range(cfg.B):
            Z = _window_Z(cube_local, cfg, d0 + dl, b, bin0, nbins)
            Y[dl][:, b * cfg.K:(b + 1) * cfg.K] = np.conj(W[dl, b].astype(np.complex128)) @ Z
    return Y


def _rand_c64(rng, shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64)


def test_apply_hand_n2():
    """hand_n2.json: w = (1/2 + i/8, 1/2 - i/8) applied to z_0 = (1, i), z_1 = (1, -1) gives
    Y = (3/8 + 3i/8, -i/4) (worked by hand in the fixture's derivation)."""
    with open(os.path.join(GOLDEN, "hand_n2.json")) as f:
        g = json.load(f)
    p = g["params"]
    cube = (np.array(g["cube_re"]) + 1j * np.array(g["cube_im"])).astype(np.complex64)
    W = (np.array(g["W_re"]) + 1j * np.array(g["W_im"])).astype(np.complex64)
    Yexp = np.array(g["Y_re"]) + 1j * np.array(g["Y_im"])
    op = OracleParams(p["C"], p["T"], p["D"], p["R"], p["K"], p["S"], p["lam"])
    Y = oracle.apply(op, cube, W.reshape(1, 1, p["S"], p["C"] * p["T"]))
    assert np.array_equal(Y[0], Yexp)  # every value is a dyadic rational: exact


def test_apply_vs_numpy_definition():
    rng = np.random.default_rng(11)
    for cfg in (synth.CONFIGS["tiny"], synth.CONFIGS["small"].with_(D=6, R=96),
                synth.CONFIGS["medium"].with_(D=7, R=128)):
        cube = synth.datacube(cfg)
        W = _rand_c64(rng, (cfg.D, cfg.B, cfg.S, cfg.N))
        op = OracleParams(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam)
        Y = oracle.apply(op, cube, W)
        Yn = _numpy_apply(cube, W, cfg, 0, cfg.D, 0, cfg.D)
        assert np.abs(Y - Yn).max() <= 1e-12 * np.abs(Yn).max(), cfg.name


def test_apply_shard_offsets_vs_numpy():
    """A shard whose window wraps the cube edge: dop_begin = 0, cube_bin0 = D - h (reading r-2),
    and an interior shard; the W32 / Y rows are the shard's local ones."""
    rng = np.random.default_rng(12)
    cfg = synth.CONFIGS["small"].with_(D=16, R=64)
    full = synth.datacube(cfg)
    for lo, cnt in ((0, 3), (5, 4), (cfg.D - 2, 2)):
        b0, nb = synth.shard_window(cfg, lo, cnt)
        local = np.ascontiguousarray(full[(b0 + np.arange(nb)) % cfg.D])
        W = _rand_c64(rng, (cnt, cfg.B, cfg.S, cfg.N))
        op = OracleParams(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam, dop_begin=lo, dop_count=cnt,
                          cube_bin0=b0, cube_bins=nb)
        Y = oracle.apply(op, local, W)
        Yn = _numpy_apply(local, W, cfg, lo, cnt, b0, nb)
        assert np.abs(Y - Yn).max() <= 1e-12 * np.abs(Yn).max(), (lo, cnt)
        # the same weights placed in a full-cube call give the same rows
        Wf = np.zeros((cfg.D, cfg.B, cfg.S, cfg.N), np.complex64)
        Wf[lo:lo + cnt] = W
        Yf = oracle.apply(OracleParams(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), full, Wf)
        assert np.array_equal(Y, Yf[lo:lo + cnt])


def test_solve_complex64_entry_equals_promoted_f64():
    """stap_oracle_solve (complex64 in) == stap_oracle_solve_f64 on the exactly promoted bytes."""
    rng = np.random.default_rng(13)
    for N, S, cnt in ((1, 1, 3), (4, 4, 5), (12, 16, 7), (56, 16, 3)):
        A = _rand_c64(rng, (cnt, N, 2 * N))
        R64 = np.einsum("uij,ukj->uik", A.astype(np.complex128), np.conj(A.astype(np.complex128))) / (2 * N)
        R64 += 0.05 * np.eye(N)
        R32 = R64.astype(np.complex64)
        st = _rand_c64(rng, (S, N))
        W1, g1, i1 = oracle.solve(R32, st)
        W2, g2, i2 = oracle.solve(R32.astype(np.complex128), st.astype(np.complex128))
        assert np.array_equal(W1, W2) and np.array_equal(g1, g2) and np.array_equal(i1, i2)
        # MVDR definition with an independent solver (numpy LAPACK gesv), reading c-9
        Rp = R32.astype(np.complex128)
        for u in range(cnt):
            V = np.linalg.solve(Rp[u], st.astype(np.complex128).T).T  # [S][N]
            gam = np.einsum("kn,kn->k", np.conj(st.astype(np.complex128)), V).real
            kappa = np.linalg.cond(Rp[u])
            assert np.abs(g1[u] - gam).max() <= 1e-12 * kappa * np.abs(gam).max()
            assert np.abs(W1[u] - V / gam[:, None]).max() <= 1e-12 * kappa * np.abs(W1[u]).max()
        assert np.all(i1 == 0)


def test_solve_complex64_entry_info_paths():
    """Clear-cut failures through the complex64 entry: a zero matrix (pivot 1 fails -> info 1,
    W = 0) and a zero steering vector (gamma = 0 -> info = -(k+1), that k's W = 0)."""
    N, S = 6, 3
    R = np.zeros((2, N, N), np.complex64)
    R[1] = np.eye(N)
    st = np.ones((S, N), np.complex64)
    st[1] = 0
    W, g, info = oracle.solve(R, st)
    assert info[0] == 1 and np.all(W[0] == 0)
    assert info[1] == -2 and np.all(W[1, 1] == 0)
    assert np.allclose(W[1, 0], st[0] / N) and np.allclose(W[1, 2], st[2] / N)

"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle, element by
element on identical seeded complex64 inputs (-m gpu).

Tolerances:
  Y per output vector (one (d, k) range line): rel-L2 <= 1e-3   (BASELINE.json north_star)
  W per (unit, k): rel-L2 <= 1e-3; gamma: rel <= 1e-3
  R per unit (Frobenius): rel <= 1e-5 (a K-term FP32 sum, no conditioning amplification)
  apply on given weights: rel-L2 <= 1e-5 per output vector
  info: bit-exact (both sides decide on pivot > 0 / finite; only clear-cut cases are tested)
"""
import os

import numpy as np
import pytest

import oracle
import synth
from oracle import OracleParams

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def stap(cuda_ok):
    import __graft_entry__ as g
    g.build_lib()
    import paper_2203_06233_b200 as p
    return p


NT = max(1, (os.cpu_count() or 1))


def OP(cfg, **kw):
    return OracleParams(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam, **kw)


def plan_for(stap, cfg, **kw):
    return stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), device=0, **kw)


def rel_lines(Yg, Yr):
    """rel-L2 per output vector (last axis)."""
    num = np.linalg.norm(Yg - Yr, axis=-1)
    den = np.linalg.norm(Yr, axis=-1)
    return num / np.maximum(den, 1e-30)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda(0)


def run_gpu(stap, cfg, cube, st, staged=False, **kw):
    plan = plan_for(stap, cfg, **kw)
    dc = dev(cube).reshape(plan.cube_shape)
    ds = dev(st)
    if staged:
        cov = plan.covariance(dc)
        w, g, info = plan.solve_weights(cov, ds)
        y = plan.apply(dc, w)
        torch.cuda.synchronize()
        return plan, y.cpu().numpy(), info.cpu().numpy(), cov.cpu().numpy(), w.cpu().numpy(), g.cpu().numpy()
    y, info = plan.run(dc, ds)
    torch.cuda.synchronize()
    return plan, y.cpu().numpy(), info.cpu().numpy()


# ---------------------------------------------------------------- whole path vs oracle
@pytest.mark.parametrize("prec", ["fp32", "tf32x3"])
@pytest.mark.parametrize("name", ["tiny", "small", "medium"])
@pytest.mark.parametrize("mode", ["run-auto", "run-fused", "run-staged", "stages"])
def test_run_vs_oracle_full(stap, name, mode, prec):
    cfg = synth.CONFIGS[name]
    cube = synth.datacube(cfg)
    st = synth.steering(cfg, "ula" if name != "tiny" else "random")
    ref = oracle.run(OP(cfg), cube, st, nthreads=NT)
    staged = mode == "stages"
    path = mode[4:] if mode.startswith("run-") else "auto"
    if name == "tiny" and path == "fused":  # below the fused kernel's occupancy floor
        with pytest.raises(stap.StapError):
            plan_for(stap, cfg, path="fused", precision=prec)
        return
    res = run_gpu(stap, cfg, cube, st, staged=staged, path=path, precision=prec)
    assert res[0].description.startswith({"fused": "fused", "staged": "staged"}.get(path, ""))
    Y, info = res[1][0], res[2][0]
    err = rel_lines(Y, ref["Y"])
    assert np.array_equal(info, ref["info"])
    assert err.max() <= 1e-3, (name, staged, err.max(), res[0].description)


@pytest.mark.parametrize("prec", ["fp32", "tf32x3"])
@pytest.mark.parametrize("name", ["medium", "large"])
def test_run_full_size_every_bin(stap, name, prec):
    """Full BASELINE size on the GPU in the bench's launch configuration (AUTO path, the
    bench's batch of distinct cubes) against the oracle on EVERY Doppler bin, block and
    steering vector of cube 0 (OpenMP over bins; ~10-30 s of host time at large)."""
    cfg = synth.CONFIGS[name]
    M = {"medium": 16, "large": 2}[name]
    cubes = np.stack([synth.datacube(cfg, i) for i in range(M)])
    st = synth.steering(cfg, "ula")
    plan, Y, info = run_gpu(stap, cfg, cubes, st, batch=M, precision=prec)
    assert ("tcgen05" in plan.description) == (prec == "tf32x3"), plan.description
    ref = oracle.run(OP(cfg), cubes[0], st, nthreads=NT)
    err = rel_lines(Y[0], ref["Y"])
    assert np.array_equal(info[0], ref["info"])
    assert err.max() <= 1e-3, (name, err.max(), plan.description)
    # the last cube of the batch too, on sampled bins (edges + interior)
    for d in (0, cfg.D // 3, cfg.D - 1):
        b0, nb = synth.shard_window(cfg, d, 1)
        local = np.ascontiguousarray(cubes[M - 1][(b0 + np.arange(nb)) % cfg.D])
        r1 = oracle.run(OP(cfg, dop_begin=d, dop_count=1, cube_bin0=b0, cube_bins=nb), local, st, nthreads=NT)
        assert np.array_equal(info[M - 1, d], r1["info"][0])
        assert rel_lines(Y[M - 1, d], r1["Y"][0]).max() <= 1e-3, (name, d)


@pytest.mark.parametrize("split,name,G", [("weak", "large", 2), ("weak", "large", 4), ("strong", "medium", 2),
                                          ("strong", "medium", 4), ("strong", "large", 4)])
def test_shard_plans_as_bench_builds_them(stap, split, name, G):
    """The exact shard plans bench.py builds at --gpus G (bench.shard_plan_args):
    weak (BASELINE configs[4]): global D = D_cfg*G, rank g owns [g D_cfg, (g+1) D_cfg);
    strong (configs[2] "medium on 1/2/4/8"): the config's D bins split D/G per rank.  Each rank's
    buffer holds its bins plus the T-1 halo (wrapped at the ends); batch 2, precision tf32x3.
    Every rank's Y equals the unsharded run over the whole global cube bitwise (P15), and
    sampled bins at the shard edges match the oracle.  Random device data: the check is the
    shard mechanics."""
    import bench
    base = synth.CONFIGS[name]
    M = 2
    gcfg = bench.shard_plan_args(base, G, 0, split)[0]
    gen = torch.Generator(device="cuda:0").manual_seed(100 + G)
    full = torch.randn((M, gcfg.D, gcfg.C, gcfg.R), dtype=torch.complex64, device="cuda:0", generator=gen)
    st = dev(synth.steering(base, "ula"))
    pf = plan_for(stap, gcfg, batch=M, precision="tf32x3")
    Yf, If = pf.run(full, st)
    torch.cuda.synchronize()
    covered = 0
    for g in range(G):
        gc, lo, cnt, b0, nb = bench.shard_plan_args(base, G, g, split)
        assert gc.D == gcfg.D
        covered += cnt
        idx = torch.from_numpy((b0 + np.arange(nb)) % gcfg.D).cuda(0)
        local = full.index_select(1, idx).contiguous()
        ps = plan_for(stap, gcfg, dop_begin=lo, dop_count=cnt, cube_bin0=b0, cube_bins=nb, batch=M,
                      precision="tf32x3")
        assert ps.description == pf.description or split == "strong"
        assert bench.plan_shape_out(stap, ps.dims, lo, cnt, b0, nb, M) == ps.out_shape
        Ys, Is = ps.run(local, st)
        torch.cuda.synchronize()
        assert torch.equal(Ys, Yf[:, lo:lo + cnt]) and torch.equal(Is, If[:, lo:lo + cnt]), g
        if g in (0, G - 1):
            xl = local[0].cpu().numpy()
            for d in (lo, lo + cnt - 1):
                ob0, onb = synth.shard_window(gcfg, d, 1)
                rows = [(a - b0) % gcfg.D for a in (ob0 + np.arange(onb))]
                r1 = oracle.run(OP(gcfg, dop_begin=d, dop_count=1, cube_bin0=ob0, cube_bins=onb),
                                np.ascontiguousarray(xl[rows]), st.cpu().numpy(), nthreads=NT)
                assert rel_lines(Ys[0, d - lo].cpu().numpy(), r1["Y"][0]).max() <= 1e-3, (g, d)
    assert covered == gcfg.D


# ---------------------------------------------------------------- stages vs oracle
@pytest.mark.parametrize("prec", ["fp32", "tf32x3"])
@pytest.mark.parametrize("name", ["tiny", "small", "medium"])
def test_covariance_vs_oracle(stap, name, prec):
    cfg = synth.CONFIGS[name]
    cube = synth.datacube(cfg)
    if name == "medium":
        cfg2 = cfg
        Rref, _ = oracle.covariance(OP(cfg2, dop_begin=0, dop_count=24), cube)
    else:
        Rref, _ = oracle.covariance(OP(cfg), cube)
    plan = plan_for(stap, cfg, precision=prec)
    cov = plan.covariance(dev(cube).reshape(plan.cube_shape)).cpu().numpy()[0]
    cov = cov[:Rref.shape[0]]
    num = np.linalg.norm((cov - Rref).reshape(cov.shape[0], cfg.B, -1), axis=-1)
    den = np.linalg.norm(Rref.reshape(cov.shape[0], cfg.B, -1), axis=-1)
    assert (num / den).max() <= 1e-5
    # exact Hermitian mirror and real diagonal
    assert np.array_equal(cov, np.conj(np.swapaxes(cov, -1, -2)))
    assert np.all(np.diagonal(cov, axis1=-2, axis2=-1).imag == 0)


def test_covariance_large_tc_vs_oracle(stap):
    """The tcgen05 covariance at the large shape (N = 56), on a D that has wrapped edge tiles."""
    cfg = synth.CONFIGS["large"].with_(D=40, R=1024)
    cube = synth.datacube(cfg)
    Rref, _ = oracle.covariance(OP(cfg), cube)
    plan = plan_for(stap, cfg, path="staged", precision="tf32x3")
    assert "cov(tcgen05" in plan.description
    cov = plan.covariance(dev(cube).reshape(plan.cube_shape)).cpu().numpy()[0]
    num = np.linalg.norm((cov - Rref).reshape(cfg.D, cfg.B, -1), axis=-1)
    den = np.linalg.norm(Rref.reshape(cfg.D, cfg.B, -1), axis=-1)
    assert (num / den).max() <= 1e-5
    assert np.array_equal(cov, np.conj(np.swapaxes(cov, -1, -2)))
    assert np.all(np.diagonal(cov, axis1=-2, axis2=-1).imag == 0)


@pytest.mark.parametrize("name", ["medium", "large"])
@pytest.mark.parametrize("lam", [1e-2, 1e-3])
def test_tensor_core_path_vs_oracle_lambda(stap, name, lam):
    """SURVEY 8(f) NEXT-4 pin: the 3xTF32 tcgen05 covariance + apply path (staged) against
    the fp64 oracle at lambda = 1e-2 and 1e-3 (a lighter loading amplifies the R error)."""
    cfg = synth.CONFIGS[name].with_(D=24, lam=lam)
    if name == "large":
        cfg = cfg.with_(R=1024)
    cube = synth.datacube(cfg)
    st = synth.steering(cfg, "ula")
    plan = plan_for(stap, cfg, path="staged", precision="tf32x3")
    assert "cov(tcgen05" in plan.description and "apply(tcgen05" in plan.description
    ref = oracle.run(OP(cfg), cube, st, nthreads=NT)
    y, info = plan.run(dev(cube).reshape(plan.cube_shape), dev(st))
    Y, I = y.cpu().numpy()[0], info.cpu().numpy()[0]
    assert np.array_equal(I, ref["info"])
    assert rel_lines(Y, ref["Y"]).max() <= 1e-3


@pytest.mark.parametrize("name,prec", [("small", "fp32"), ("medium", "fp32"), ("medium", "tf32x3")])
def test_covariance_batch_bitwise(stap, name, prec):
    """A batched covariance equals each cube's own (every tile of every cube, incl. wrapped ones)."""
    cfg = synth.CONFIGS[name]
    M = 6
    xs = np.stack([synth.datacube(cfg, i) for i in range(M)])
    pb = plan_for(stap, cfg, batch=M, path="staged", precision=prec)
    p1 = plan_for(stap, cfg, path="staged", precision=prec)
    cb = pb.covariance(dev(xs).reshape(pb.cube_shape)).cpu().numpy()
    for n in range(M):
        c1 = p1.covariance(dev(xs[n:n + 1]).reshape(p1.cube_shape)).cpu().numpy()[0]
        assert np.array_equal(cb[n], c1), n


@pytest.mark.parametrize("name", ["tiny", "small", "medium", "large"])
def test_solve_vs_oracle(stap, name):
    """K2 fed the GPU's own complex64 covariance; the oracle solves the same bytes."""
    cfg = synth.CONFIGS[name]
    nd = min(cfg.D, 16)
    sub = cfg.with_(D=max(nd, cfg.T))
    cube = synth.datacube(sub)
    st = synth.steering(sub, "random")
    plan = plan_for(stap, sub)
    dc = dev(cube).reshape(plan.cube_shape)
    cov = plan.covariance(dc)
    w, g, info = plan.solve_weights(cov, dev(st))
    torch.cuda.synchronize()
    cov_h = cov.cpu().numpy()
    Wr, gr, ir = oracle.solve(cov_h, st)
    assert np.array_equal(info.cpu().numpy(), ir)
    e = rel_lines(w.cpu().numpy(), Wr)
    assert e.max() <= 1e-3, e.max()
    assert (np.abs(g.cpu().numpy() - gr) / gr).max() <= 1e-3
    # distortionless response in FP32
    W = w.cpu().numpy().astype(np.complex128)
    resp = np.einsum("...kn,kn->...k", W.conj(), st.astype(np.complex128))
    assert np.abs(resp - 1).max() <= 1e-4


@pytest.mark.parametrize("prec", ["fp32", "tf32x3"])
@pytest.mark.parametrize("name", ["tiny", "small", "medium", "large"])
def test_apply_vs_oracle(stap, name, prec):
    cfg = synth.CONFIGS[name]
    sub = cfg.with_(D=min(cfg.D, 8) if cfg.D > 8 else cfg.D)
    cube = synth.datacube(sub)
    rng = np.random.default_rng(1)
    W = (rng.standard_normal((sub.D, sub.B, sub.S, sub.N)) + 1j * rng.standard_normal((sub.D, sub.B, sub.S, sub.N))
         ).astype(np.complex64)
    plan = plan_for(stap, sub, precision=prec)
    y = plan.apply(dev(cube).reshape(plan.cube_shape), dev(W).reshape(plan.weights_shape)).cpu().numpy()[0]
    Yr = oracle.apply(OP(sub), cube, W)
    assert rel_lines(y, Yr).max() <= 1e-5


# ---------------------------------------------------------------- closed forms through the GPU
def test_E1_identity_covariance_gpu(stap):
    """DFT-white cube: Rhat = I => w_k = s_k/||s_k||^2 and Y = s_k^H z / ||s_k||^2 (north_star pin)."""
    cfg = synth.CONFIGS["small"]
    cube = synth.cube_e1(cfg)
    st = synth.steering(cfg, "random")
    _, Y, info = run_gpu(stap, cfg, cube, st)
    s = st.astype(np.complex128)
    wexp = s / np.sum(np.abs(s) ** 2, axis=1, keepdims=True)
    for d in (0, 7, cfg.D - 1):
        Z = np.concatenate([cube[(d - cfg.h + t) % cfg.D] for t in range(cfg.T)], 0).astype(np.complex128)
        assert rel_lines(Y[0, d], wexp.conj() @ Z).max() <= 1e-5
    assert np.all(info == 0)


def test_E3_target_gpu(stap):
    cfg = synth.CONFIGS["small"]
    cube = synth.datacube(cfg)
    rng = np.random.default_rng(3)
    st = (rng.integers(-3, 4, (cfg.S, cfg.N)) + 1j * rng.integers(-3, 4, (cfg.S, cfg.N))).astype(np.complex64)
    st[:, 0] += 4
    alpha = 3 - 2j
    picks = [(0, 5, 1), (100, 77, 0), (cfg.D - 1, 511, 15)]
    for d, r, k in picks:
        for t in range(cfg.T):
            cube[(d - cfg.h + t) % cfg.D, :, r] = alpha * st[k, t * cfg.C:(t + 1) * cfg.C]
    _, Y, _ = run_gpu(stap, cfg, cube, st)
    for d, r, k in picks:
        assert abs(Y[0, d, k, r] - alpha) <= 1e-4 * abs(alpha)


def test_path_and_precision_selection(stap):
    """path=fused on a shape the fused kernel cannot hold is STAP_ERR_UNSUPPORTED; AUTO picks
    staged there.  The tensor-core stages run only under precision=tf32x3 (explicit opt-in)."""
    cfg = synth.CONFIGS["large"]
    with pytest.raises(stap.StapError) as e:
        plan_for(stap, cfg, path="fused")
    assert e.value.code == 3
    dl = plan_for(stap, cfg).description
    assert dl.startswith("staged") and "tcgen05" not in dl, dl
    dl = plan_for(stap, cfg, precision="tf32x3").description
    assert dl.startswith("staged") and "cov(tcgen05" in dl and "apply(tcgen05" in dl, dl
    dm = plan_for(stap, synth.CONFIGS["medium"], precision="tf32x3").description
    assert dm.startswith("staged") and "cov(tcgen05" in dm and "apply(tcgen05" in dm
    assert "tcgen05" not in plan_for(stap, synth.CONFIGS["medium"], path="staged").description
    assert plan_for(stap, synth.CONFIGS["medium"], path="fused").description.startswith("fused")
    assert plan_for(stap, synth.CONFIGS["small"]).description.startswith("fused")
    assert plan_for(stap, synth.CONFIGS["small"], precision="tf32x3").description.startswith("fused")


def test_plan_as_first_cuda_call(stap):
    """A plan created before any other CUDA call in a fresh process selects the same kernels as
    any later plan (the tcgen05 stages depend on a driver tensor-map encode, which needs the
    primary context: stap_plan_create creates it).  Round 2 found a first plan silently on the
    SIMT covariance and apply."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import synth, paper_2203_06233_b200 as p\n"
            "c = synth.CONFIGS['large']\n"
            "print(p.StapPlan(p.Dims(c.C, c.T, c.D, c.R, c.K, c.S, c.lam), precision='tf32x3').description)")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300,
                         check=True).stdout
    assert "cov(tcgen05" in out and "apply(tcgen05" in out, out


# ---------------------------------------------------------------- composition, shards, batch, determinism
@pytest.mark.parametrize("name", ["small", "medium"])
def test_fused_equals_staged(stap, name):
    cfg = synth.CONFIGS[name]
    cube = synth.datacube(cfg)
    st = synth.steering(cfg, "ula")
    pf, Yf, If = run_gpu(stap, cfg, cube, st, path="fused")
    assert pf.description.startswith("fused")
    # same arithmetic: the staged path at the default FP32 precision (SIMT covariance and apply)
    res = run_gpu(stap, cfg, cube, st, staged=True, path="staged")
    assert "cov(simt" in res[0].description and "apply(simt" in res[0].description
    assert np.array_equal(If, res[2])
    e = rel_lines(Yf, res[1]).max()
    assert e <= 1e-5, e
    # the default staged path (tcgen05 3xTF32 covariance and apply where they apply) agrees
    # within the oracle tolerance: R differs by <= ~2e-6 relative, amplified at most by
    # the loaded condition number (<= N / lambda); the apply adds <= ~1e-6 per line
    res2 = run_gpu(stap, cfg, cube, st, staged=True, path="staged", precision="tf32x3")
    assert np.array_equal(If, res2[2])
    assert rel_lines(Yf, res2[1]).max() <= 1e-3


@pytest.mark.parametrize("name,G,prec", [("tiny", 3, "fp32"), ("small", 2, "fp32"), ("small", 8, "fp32"),
                                         ("medium", 4, "fp32"), ("medium", 4, "tf32x3")])
def test_doppler_shards_bitwise(stap, name, G, prec):
    """P15: every shard plan on a slice+halo buffer reproduces the full run bitwise."""
    cfg = synth.CONFIGS[name]
    cube = synth.datacube(cfg)
    st = synth.steering(cfg, "ula")
    _, Yfull, Ifull = run_gpu(stap, cfg, cube, st, precision=prec)
    for g in range(G):
        lo, cnt = synth.shard_range(cfg.D, G, g)
        b0, nb = synth.shard_window(cfg, lo, cnt)
        local = np.ascontiguousarray(cube[(b0 + np.arange(nb)) % cfg.D])
        _, Y, I = run_gpu(stap, cfg, local, st, dop_begin=lo, dop_count=cnt, cube_bin0=b0, cube_bins=nb,
                          precision=prec)
        assert np.array_equal(Y[0], Yfull[0, lo:lo + cnt])
        assert np.array_equal(I[0], Ifull[0, lo:lo + cnt])


def test_batch_bitwise(stap):
    cfg = synth.CONFIGS["small"]
    cubes = np.stack([synth.datacube(cfg, i) for i in range(3)])
    st = synth.steering(cfg, "ula")
    _, Yb, Ib = run_gpu(stap, cfg, cubes, st, batch=3)
    for i in range(3):
        _, Y1, I1 = run_gpu(stap, cfg, cubes[i], st)
        assert np.array_equal(Yb[i], Y1[0]) and np.array_equal(Ib[i], I1[0])


def test_determinism_and_immutability(stap):
    cfg = synth.CONFIGS["small"]
    cube = synth.datacube(cfg)
    st = synth.steering(cfg, "ula")
    plan = plan_for(stap, cfg)
    dc = dev(cube).reshape(plan.cube_shape)
    ds = dev(st)
    c0, s0 = dc.clone(), ds.clone()
    y1, i1 = plan.run(dc, ds)
    y2, i2 = plan.run(dc, ds)
    plan.solve_weights(plan.covariance(dc), ds)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2) and torch.equal(i1, i2)
    assert torch.equal(dc, c0) and torch.equal(ds, s0)


def test_run_host_matches_device(stap):
    cfg = synth.CONFIGS["small"]
    cube = synth.datacube(cfg)
    st = synth.steering(cfg, "ula")
    plan = plan_for(stap, cfg)
    _, Yd, Id = run_gpu(stap, cfg, cube, st)
    hc = torch.from_numpy(cube).pin_memory()
    hs = torch.from_numpy(st).pin_memory()
    ho = torch.empty(plan.out_shape, dtype=torch.complex64).pin_memory()
    hi = torch.empty(plan.info_shape, dtype=torch.int32).pin_memory()
    ws = torch.empty(plan.host_workspace_bytes, dtype=torch.uint8, device="cuda:0")
    plan.run_host(hc, hs, ho, hi, ws)
    torch.cuda.synchronize()
    assert np.array_equal(ho.numpy(), Yd) and np.array_equal(hi.numpy(), Id)


@pytest.mark.parametrize("name,M", [("small", 8), ("medium", 4), ("large", 2), ("odd-info", 2), ("odd-info", 6)])
def test_run_host_pipelined_batch(stap, name, M):
    """Batched stap_run_host (chunked, copies overlapped on internal streams) == device stap_run.
    "odd-info": one cube's info block is 24 bytes (D = 2, B = 3), so no chunk count keeps
    16-byte chunk offsets and the call runs unchunked (plan creation once failed there)."""
    if name == "odd-info":
        cfg = synth.CONFIGS["tiny"].with_(D=2, R=18, K=6, C=3, T=2)
    else:
        cfg = synth.CONFIGS[name]
    if name not in ("small", "odd-info"):
        cfg = cfg.with_(D=32)
    xs = np.stack([synth.datacube(cfg, i) for i in range(M)])
    st = synth.steering(cfg, "ula")
    plan = plan_for(stap, cfg, batch=M)
    yd, idv = plan.run(dev(xs).reshape(plan.cube_shape), dev(st))
    hc = torch.from_numpy(xs).pin_memory()
    hs = torch.from_numpy(st).pin_memory()
    ho = torch.full(plan.out_shape, float("nan"), dtype=torch.complex64).pin_memory()
    hi = torch.full(plan.info_shape, -7, dtype=torch.int32).pin_memory()
    ws = torch.empty(plan.host_workspace_bytes, dtype=torch.uint8, device="cuda:0")
    for _ in range(2):  # twice: the second call must order after the first
        plan.run_host(hc, hs, ho, hi, ws)
        torch.cuda.synchronize()
        assert np.array_equal(ho.numpy(), yd.cpu().numpy()) and np.array_equal(hi.numpy(), idv.cpu().numpy())


# ---------------------------------------------------------------- edge and degenerate cases
@pytest.mark.parametrize("kw", [
    dict(C=1, T=1, D=1, R=8, K=2, S=1),        # N = 1, D = T = 1
    dict(C=8, T=8, D=8, R=64, K=32, S=32),     # maximum N = 64, S = 32
    dict(C=3, T=5, D=5, R=24, K=6, S=3),       # D = T, odd C, odd S, K < N (loading keeps R PD)
    dict(C=6, T=5, D=37, R=128, K=64, S=16),   # ragged bin runs
    dict(C=5, T=2, D=11, R=40, K=4, S=7),      # C without a fused specialisation -> staged path
    dict(C=2, T=4, D=9, R=32, K=16, S=5),      # even T (h = 1)
    # tensor-core stages (cov_tc: K % 16 == 0, 24 <= N <= 64; apply_tc: S == 16, K % 64 == 0)
    dict(C=8, T=8, D=8, R=128, K=64, S=16),    # N = 64 on both tcgen05 stages
    dict(C=6, T=4, D=4, R=1024, K=1024, S=16), # N = 24 (smallest tc N), K = 1024 (largest), B = 1, D = T
    dict(C=3, T=8, D=50, R=128, K=128, S=16),  # C = 3: a Gram tile of 42 bins (126 of 128 rows)
    dict(C=7, T=9, D=13, R=192, K=64, S=16),   # odd N = 63, ragged tiles
    dict(C=5, T=5, D=67, R=64, K=64, S=16),    # odd N = 25, prime D (wrapped edge tiles)
    dict(C=3, T=9, D=9, R=48, K=16, S=16),     # cov_tc at K = 16, SIMT apply (K % 64 != 0)
    # every chol.cuh instantiation family: N = 13..24 (4x4 lanes, two matrices per warp),
    # N = 25..32 (4x8 lanes), S > 16 there, N = 33 with S <= 8 (14x7 blocks, one
    # RHS column per lane), N = 48 with S = 32 (8x8 lanes)
    dict(C=1, T=13, D=15, R=64, K=32, S=8),    # N = 13: the smallest N on chol.cuh
    dict(C=4, T=4, D=9, R=128, K=64, S=16),    # N = 16, S = 16
    dict(C=2, T=7, D=11, R=64, K=32, S=32),    # N = 14, S = 32
    dict(C=1, T=17, D=19, R=64, K=32, S=3),    # N = 17 (4x4 lanes, 6x6 blocks)
    dict(C=5, T=5, D=9, R=64, K=32, S=16),     # N = 25: the first N on 4x8 lanes, 8x4 blocks
    dict(C=4, T=5, D=7, R=96, K=48, S=24),     # N = 20, S = 24 (four RHS columns per lane)
    dict(C=3, T=11, D=13, R=128, K=64, S=8),   # N = 33, S = 8 (40-row layout)
    dict(C=8, T=5, D=9, R=128, K=64, S=16),    # N = 40, S = 16
    dict(C=7, T=6, D=11, R=64, K=32, S=5),     # N = 42, S = 5 (48-row layout)
    dict(C=7, T=7, D=9, R=128, K=64, S=16),    # N = 49, S = 16 (56-row layout)
    dict(C=8, T=6, D=9, R=128, K=128, S=32),   # N = 48, S = 32
])
@pytest.mark.parametrize("staged,prec", [(False, "fp32"), (True, "fp32"), (True, "tf32x3")])
def test_edge_shapes(stap, kw, staged, prec):
    cfg = synth.StapConfig("edge", lam=1e-2, cfg_id=7, **kw)
    cube = synth.datacube(cfg)
    st = synth.steering(cfg, "random")
    ref = oracle.run(OP(cfg), cube, st, nthreads=NT)
    res = run_gpu(stap, cfg, cube, st, staged=staged, precision=prec)
    assert np.array_equal(res[2][0], ref["info"])
    assert rel_lines(res[1][0], ref["Y"]).max() <= 1e-3


@pytest.mark.parametrize("name", ["small", "medium", "large"])
@pytest.mark.parametrize("staged,prec", [(False, "fp32"), (True, "fp32"), (True, "tf32x3")])
def test_info_paths(stap, name, staged, prec):
    cfg = {"medium": synth.CONFIGS["medium"].with_(D=24),
           "large": synth.CONFIGS["large"].with_(D=16, R=512)}.get(name, synth.CONFIGS[name])
    cube = synth.datacube(cfg)
    st = synth.steering(cfg, "random")
    cube[:, :, cfg.K:2 * cfg.K] = 0          # block 1 zero everywhere -> info = 1
    st[5] = 0                                 # steering 5 zero -> info = -6 elsewhere
    ref = oracle.run(OP(cfg), cube, st, nthreads=NT)
    res = run_gpu(stap, cfg, cube, st, staged=staged, precision=prec)
    Y, info = res[1][0], res[2][0]
    assert np.array_equal(info, ref["info"])
    assert np.all(info[:, 1] == 1) and np.all(info[:, 0] == -6)
    assert np.all(Y[:, :, cfg.K:2 * cfg.K] == 0) and np.all(Y[:, 5] == 0)
    good = np.ones(Y.shape[:2], bool)
    good[:, 5] = False
    mask = np.ones(cfg.R, bool)
    mask[cfg.K:2 * cfg.K] = False
    assert rel_lines(Y[good][:, mask], ref["Y"][good][:, mask]).max() <= 1e-3


def test_bad_pointer_alignment(stap):
    cfg = synth.CONFIGS["tiny"]
    plan = plan_for(stap, cfg)
    buf = torch.zeros(plan.out_shape[1] * cfg.S * cfg.R * 2 + 8, dtype=torch.float32, device="cuda:0")
    with pytest.raises(stap.StapError) as e:
        stap.stap_covariance(plan.handle, buf.data_ptr() + 8, buf.data_ptr(), None)
    assert e.value.code == 4


# ---------------------------------------------------------------- race / stability stress (compute-sanitizer is closed on this pool)
@pytest.mark.parametrize("prec", ["fp32", "tf32x3"])
@pytest.mark.parametrize("name", ["tiny", "small", "medium", "large"])
def test_repeat_runs_bitwise(stap, name, prec):
    """Shared-memory races (mbarrier phases, aliased scratch, group barriers) show up as
    run-to-run differences: 8 repeated launches of every entry point must agree bitwise."""
    cfg = synth.CONFIGS[name]
    if name in ("medium", "large"):
        cfg = cfg.with_(D=32)
    x = np.stack([synth.datacube(cfg, i) for i in range(2)])
    st = synth.steering(cfg, "random")
    plan = plan_for(stap, cfg, batch=2, precision=prec)
    dc, ds = dev(x).reshape(plan.cube_shape), dev(st)
    y0, i0 = plan.run(dc, ds)
    c0 = plan.covariance(dc)
    w0, g0, j0 = plan.solve_weights(c0, ds)
    a0 = plan.apply(dc, w0)
    for _ in range(8):
        y, i = plan.run(dc, ds)
        c = plan.covariance(dc)
        w, g, j = plan.solve_weights(c, ds)
        a = plan.apply(dc, w)
        assert torch.equal(c, c0), "covariance"
        assert torch.equal(w, w0) and torch.equal(g, g0) and torch.equal(j, j0), "solve"
        assert torch.equal(a, a0), "apply"
        assert torch.equal(i, i0), "run info"
        assert torch.equal(y, y0), "run"



def test_wrap_only_window_shard(stap):
    """A shard whose whole window wraps around the cube edge (bins D-1, 0, 1, ...)."""
    cfg = synth.CONFIGS["small"]
    cube = synth.datacube(cfg)
    st = synth.steering(cfg, "ula")
    _, Yfull, _ = run_gpu(stap, cfg, cube, st)
    lo, cnt = 0, 3
    b0, nb = synth.shard_window(cfg, lo, cnt)
    assert b0 == cfg.D - cfg.h
    local = np.ascontiguousarray(cube[(b0 + np.arange(nb)) % cfg.D])
    _, Y, _ = run_gpu(stap, cfg, local, st, dop_begin=lo, dop_count=cnt, cube_bin0=b0, cube_bins=nb)
    assert np.array_equal(Y[0], Yfull[0, lo:lo + cnt])


# ---------------------------------------------------------------- Doppler front end
@pytest.mark.parametrize("name,kw,M", [("tiny", {}, 1), ("small", {}, 2), ("medium", dict(R=128), 1),
                                       ("large", dict(R=128), 1), ("small", dict(D=8192, R=64, K=32), 1)])
def test_doppler_vs_oracle(stap, name, kw, M):
    """K0 (stap_doppler) against the fp64 windowed DFT, per (cube, channel, cell) column over d."""
    cfg = synth.CONFIGS[name].with_(**kw)
    rng = np.random.default_rng(7)
    raw = (rng.standard_normal((M, cfg.D, cfg.C, cfg.R)) + 1j * rng.standard_normal((M, cfg.D, cfg.C, cfg.R))).astype(np.complex64)
    w = np.hanning(cfg.D + 2)[1:-1].astype(np.float32)
    plan = plan_for(stap, cfg, batch=M)
    X = plan.doppler(dev(raw).reshape(plan.cube_shape), dev(w)).cpu().numpy()
    ref = oracle.doppler(w, raw, nthreads=NT)
    err = np.linalg.norm(X - ref, axis=1) / np.linalg.norm(ref, axis=1)  # over d
    assert err.max() <= 1e-5, err.max()
    # deterministic
    X2 = plan.doppler(dev(raw).reshape(plan.cube_shape), dev(w)).cpu().numpy()
    assert np.array_equal(X, X2)


@pytest.mark.parametrize("D", [2, 4, 16, 32, 64, 128, 2048])
@pytest.mark.parametrize("R", [48, 24, 20, 18])
def test_doppler_every_split_and_tile(stap, D, R):
    """Every D = L1*L2 instantiation of the register FFT (16..128 here; 256..1024 above) and
    its tile widths RC = 16 / 8 / 4 (R = 48 / 24 / 20), plus the shared-memory fallback (R = 18:
    no RC >= 4 divides it; D = 2, 4, 2048 are outside the register path), vs the fp64 DFT."""
    cfg = synth.CONFIGS["tiny"].with_(D=D, R=R, C=3, T=2, K=R // 2 if R % 4 == 0 else 6)  # K even
    rng = np.random.default_rng(D * 100 + R)
    raw = (rng.standard_normal((2, D, cfg.C, R)) + 1j * rng.standard_normal((2, D, cfg.C, R))).astype(np.complex64)
    w = (0.5 + rng.random(D)).astype(np.float32)
    plan = plan_for(stap, cfg, batch=2)
    X = plan.doppler(dev(raw).reshape(plan.cube_shape), dev(w)).cpu().numpy()
    ref = oracle.doppler(w, raw, nthreads=NT)
    err = np.linalg.norm(X - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert err.max() <= 1e-5, err.max()


def test_doppler_front_end_feeds_the_path(stap):
    """raw -> stap_doppler -> stap_run equals the oracle chain doppler -> run (within the Y tolerance)."""
    cfg = synth.CONFIGS["small"].with_(D=64)
    rng = np.random.default_rng(8)
    raw = (rng.standard_normal((cfg.D, cfg.C, cfg.R)) + 1j * rng.standard_normal((cfg.D, cfg.C, cfg.R))).astype(np.complex64)
    w = np.hanning(cfg.D + 2)[1:-1].astype(np.float32)
    st = synth.steering(cfg, "ula")
    plan = plan_for(stap, cfg)
    cube = plan.doppler(dev(raw).reshape(plan.cube_shape), dev(w))
    y, info = plan.run(cube, dev(st))
    ref = oracle.run(OP(cfg), plan.doppler(dev(raw).reshape(plan.cube_shape), dev(w)).cpu().numpy()[0], st, nthreads=NT)
    assert np.array_equal(info.cpu().numpy()[0], ref["info"])
    assert rel_lines(y.cpu().numpy()[0], ref["Y"]).max() <= 1e-3


def test_doppler_rejects(stap):
    cfg = synth.CONFIGS["small"]
    import torch
    w = torch.ones(cfg.D, dtype=torch.float32, device="cuda")
    b0, nb = synth.shard_window(cfg, 0, 8)
    shard = plan_for(stap, cfg, dop_begin=0, dop_count=8, cube_bin0=b0, cube_bins=nb)
    raw = torch.zeros(shard.cube_shape, dtype=torch.complex64, device="cuda")
    with pytest.raises(stap.StapError) as e:
        shard.doppler(raw, w)
    assert e.value.code == 3
    odd = synth.CONFIGS["small"].with_(D=48)
    p = plan_for(stap, odd)
    with pytest.raises(stap.StapError) as e:
        p.doppler(torch.zeros(p.cube_shape, dtype=torch.complex64, device="cuda"),
                  torch.ones(odd.D, dtype=torch.float32, device="cuda"))
    assert e.value.code == 3

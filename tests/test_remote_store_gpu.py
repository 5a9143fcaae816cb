"""The remote-store epilogue on ONE GPU (-m gpu; include/stap.h out_n_peers).

A plan with out_n_peers = 1 repeats every Y store at `out + out_peer_offset[0]`.  Pointing the
offset at a second buffer on the same device exercises exactly the store code the fused
all-gather uses across GPUs (the REMOTE instantiations of the fused, SIMT-apply and tcgen05
apply epilogues), without a second GPU: both copies must equal the plain-store plan's output
bitwise, and the oracle within the Y tolerance (1e-3 per output vector).
"""
import os

import numpy as np
import pytest

import oracle
import synth
from oracle import OracleParams

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

NT = max(1, (os.cpu_count() or 1))


@pytest.fixture(scope="module")
def stap(cuda_ok):
    import __graft_entry__ as g
    g.build_lib()
    import paper_2203_06233_b200 as p
    return p


# (config, D override, path, precision, the apply epilogue it exercises)
CASES = [
    ("tiny", None, "staged", "fp32", "apply(simt"),
    ("small", 64, "fused", "fp32", "fused"),
    ("small", 64, "staged", "fp32", "apply(simt"),
    ("medium", 24, "fused", "fp32", "fused"),
    ("medium", 24, "staged", "fp32", "apply(simt"),
    ("medium", 24, "staged", "tf32x3", "apply(tcgen05"),
    ("large", 16, "staged", "tf32x3", "apply(tcgen05"),
]


@pytest.mark.parametrize("name,D,path,prec,expect", CASES)
@pytest.mark.parametrize("entry", ["run", "apply"])
def test_peer_copy_store_one_gpu(stap, name, D, path, prec, expect, entry):
    cfg = synth.CONFIGS[name] if D is None else synth.CONFIGS[name].with_(D=D)
    if name == "large":
        cfg = cfg.with_(R=1024)
    if entry == "apply" and path == "fused":
        pytest.skip("stap_apply is a stage entry point (SIMT or tcgen05 apply), not the fused kernel")
    M = 2
    cubes = np.stack([synth.datacube(cfg, i) for i in range(M)])
    st = synth.steering(cfg, "ula")
    dims = stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam)
    plain = stap.StapPlan(dims, batch=M, device=0, path=path, precision=prec)
    dc = torch.from_numpy(cubes).cuda(0).reshape(plain.cube_shape)
    ds = torch.from_numpy(st).cuda(0)
    # one allocation holding both copies; the second at a 16-byte multiple past the first
    n = int(np.prod(plain.out_shape))
    buf = torch.empty((2 * n + 2,), dtype=torch.complex64, device="cuda:0")
    buf.view(torch.float32).fill_(float("nan"))
    y0, y1 = buf[:n].view(plain.out_shape), buf[n + 2:2 * n + 2].view(plain.out_shape)
    off = y1.data_ptr() - y0.data_ptr()
    assert off % 16 == 0
    remote = stap.StapPlan(dims, batch=M, device=0, path=path, precision=prec, out_peer_offsets=(off,))
    assert remote.description == plain.description and expect in plain.description, plain.description
    if entry == "run":
        yp, ip = plain.run(dc, ds)
        _, ir = remote.run(dc, ds, out=y0)
        assert torch.equal(ip, ir)
    else:
        w, _, ip = plain.solve_weights(plain.covariance(dc), ds)
        yp = plain.apply(dc, w)
        remote.apply(dc, w, out=y0)
    torch.cuda.synchronize()
    assert torch.equal(y0.view(torch.float32), yp.view(torch.float32))
    assert torch.equal(y1.view(torch.float32), yp.view(torch.float32))
    assert torch.isnan(buf[n:n + 2].view(torch.float32)).all()  # nothing written between the copies
    ref = oracle.run(OracleParams(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), cubes[1], st, nthreads=NT)
    Y = y1[1].cpu().numpy()
    err = np.linalg.norm(Y - ref["Y"], axis=-1) / np.linalg.norm(ref["Y"], axis=-1)
    assert err.max() <= 1e-3, err.max()


def test_remote_plan_rejects_raw_address_for_other_buffers(stap):
    """The binding accepts an int device address only as `out` of a remote-store plan."""
    cfg = synth.CONFIGS["tiny"]
    dims = stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam)
    plan = stap.StapPlan(dims, device=0)
    cube = torch.zeros(plan.cube_shape, dtype=torch.complex64, device="cuda:0")
    st = torch.zeros((cfg.S, cfg.N), dtype=torch.complex64, device="cuda:0")
    out = torch.empty(plan.out_shape, dtype=torch.complex64, device="cuda:0")
    with pytest.raises(TypeError):
        plan.run(cube, st, out=out.data_ptr())
    with pytest.raises(ValueError):
        plan.run(cube, st, out=torch.empty(3, dtype=torch.complex64, device="cuda:0"))
    with pytest.raises(ValueError):
        plan.run(cube, st, info=torch.empty(plan.info_shape, dtype=torch.int64, device="cuda:0"))

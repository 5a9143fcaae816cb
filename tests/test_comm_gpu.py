"""The C-ABI multi-GPU extension, one process driving two GPUs (-m gpu, needs 2 GPUs).

stap_comm_create over devices 0 and 1; each device runs its rank's weak Doppler shard
(BASELINE configs[4] pattern: global D = 2 x D_cfg, rank r owns [r D_cfg, (r+1) D_cfg) from a
buffer with its bins plus the T-1 halo) into its slice of out_full [2][batch][Dl][S][R];
  - stap_comm_allgather_out (in-place ncclAllGather) must leave on BOTH devices exactly the
    unsharded run's output (bitwise, P15 + the gather);
  - stap_comm_peer_offsets + plans with out_n_peers (the all-gather fused into the apply
    epilogue by peer stores) must produce the same bytes.
The one-process-per-GPU variant (stap_comm_init_rank, IPC peer mapping) runs through
bench.py --gather comm / comm-peer in test_peer_gather_gpu.py.
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def stap(cuda_ok):
    import __graft_entry__ as g
    g.build_lib()
    import paper_2203_06233_b200 as p
    return p


@pytest.mark.parametrize("name,prec", [("small", "fp32"), ("medium", "tf32x3"), ("large", "tf32x3")])
def test_comm_single_process_two_gpus(stap, name, prec):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    base = synth.CONFIGS[name]
    if name == "large":
        base = base.with_(D=64, R=1024)
    G, M = 2, 2
    gcfg = base.with_(D=base.D * G)
    dims = stap.Dims(gcfg.C, gcfg.T, gcfg.D, gcfg.R, gcfg.K, gcfg.S, gcfg.lam)
    gen = torch.Generator(device="cuda:0").manual_seed(7)
    full = torch.randn((M, gcfg.D, gcfg.C, gcfg.R), dtype=torch.complex64, device="cuda:0", generator=gen)
    st = torch.from_numpy(synth.steering(base, "ula"))
    ref = stap.StapPlan(dims, batch=M, device=0, precision=prec).run(full, st.cuda(0))[0]
    torch.cuda.synchronize(0)
    comm = stap.StapComm(devices=[0, 1])
    assert comm.nranks == 2 and comm.nlocal == 2
    cubes, plans, outs, steers = [], [], [], []
    for r in range(G):
        lo, cnt = r * base.D, base.D
        b0, nb = synth.shard_window(gcfg, lo, cnt)
        idx = torch.from_numpy((b0 + np.arange(nb)) % gcfg.D).cuda(0)
        cubes.append(full.index_select(1, idx).contiguous().to(f"cuda:{r}"))
        plans.append(stap.StapPlan(dims, dop_begin=lo, dop_count=cnt, cube_bin0=b0, cube_bins=nb, batch=M, device=r,
                                   precision=prec))
        o = torch.empty((G,) + plans[r].out_shape, dtype=torch.complex64, device=f"cuda:{r}")
        o.view(torch.float32).fill_(float("nan"))
        outs.append(o)
        steers.append(st.to(f"cuda:{r}"))
    # expected gathered layout: [rank][batch][Dl][S][R]
    expect = torch.stack([ref[:, r * base.D:(r + 1) * base.D] for r in range(G)]).cpu()

    # (1) stage outputs into the own slice, then the in-place NCCL all-gather
    for r in range(G):
        with torch.cuda.device(r):
            plans[r].run(cubes[r], steers[r], out=outs[r][r])
    comm.allgather_out(outs, plans)
    for r in range(G):
        torch.cuda.synchronize(r)
        assert torch.equal(outs[r].cpu().view(torch.float32), expect.view(torch.float32)), r

    # (2) the all-gather fused into the apply epilogue: peer-copy stores, no collective call
    offs = comm.peer_offsets(outs)
    assert all(len(o) == 1 for o in offs)
    assert comm.peer_offsets(outs) == offs  # a repeat call with the same buffers: the same offsets
    for r in range(G):
        outs[r].view(torch.float32).fill_(float("nan"))
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    fplans = [stap.StapPlan(dims, dop_begin=p.dop_begin, dop_count=p.dop_count, cube_bin0=p.cube_bin0,
                            cube_bins=p.cube_bins, batch=M, device=r, precision=prec, out_peer_offsets=offs[r])
              for r, p in enumerate(plans)]
    for r in range(G):
        with torch.cuda.device(r):
            fplans[r].run(cubes[r], steers[r], out=outs[r][r])
    for r in range(G):
        torch.cuda.synchronize(r)
    for r in range(G):
        assert torch.equal(outs[r].cpu().view(torch.float32), expect.view(torch.float32)), r

    # (3) the gather by copy engines: plain local stores, then stap_comm_push_out
    for r in range(G):
        outs[r].view(torch.float32).fill_(float("nan"))
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    for r in range(G):
        with torch.cuda.device(r):
            plans[r].run(cubes[r], steers[r], out=outs[r][r])
    comm.push_out(outs, plans)
    for r in range(G):
        torch.cuda.synchronize(r)
    for r in range(G):
        assert torch.equal(outs[r].cpu().view(torch.float32), expect.view(torch.float32)), r
    # push_out needs the buffers peer_offsets mapped
    other = [torch.empty_like(o) for o in outs]
    with pytest.raises(stap.StapError) as e:
        comm.push_out(other, plans)
    assert e.value.code == 2


def test_comm_rejects_mismatched_plans(stap):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    cfg = synth.CONFIGS["tiny"]
    comm = stap.StapComm(devices=[0, 1])
    d = stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam)
    p0 = stap.StapPlan(d, device=0, dop_begin=0, dop_count=4)
    p1 = stap.StapPlan(d, device=1, dop_begin=4, dop_count=3)  # a different slice shape
    outs = [torch.empty((2,) + p0.out_shape, dtype=torch.complex64, device=f"cuda:{r}") for r in range(2)]
    with pytest.raises(stap.StapError) as e:
        comm.allgather_out(outs, [p0, p1])
    assert e.value.code == 2

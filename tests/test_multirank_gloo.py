"""World-size-2 gloo tests of the Doppler-shard logic bench.py uses at N > 1
(-m "not gpu"): each rank builds exactly the slice + halo buffer bench.make_inputs
builds, computes its owned bins (with the oracle, on the CPU), and the gathered
result must equal the unsharded computation bitwise (pin P15; SPEC chunk rule)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import oracle
        import synth
        cfg = synth.CONFIGS["tiny"].with_(T=3, D=8)
        if mode == "weak":
            # bench's N>1 layout: global D = D_cfg * world, rank owns a D_cfg slice + halo
            gcfg, lo, cnt, b0, nb, x, st = bench.make_inputs(cfg, world, rank, cubes=1)
        else:
            # strong split of one cube by the contiguous chunk rule
            gcfg = cfg
            lo, cnt = synth.shard_range(cfg.D, world, rank)
            b0, nb = synth.shard_window(cfg, lo, cnt)
            x = synth.datacube_bins(cfg, (b0 + np.arange(nb)) % cfg.D)[None]
            st = synth.steering(cfg, "ula")
        p = oracle.OracleParams(cfg.C, cfg.T, gcfg.D, cfg.R, cfg.K, cfg.S, cfg.lam, dop_begin=lo, dop_count=cnt,
                                cube_bin0=b0, cube_bins=nb)
        Y = oracle.run(p, np.ascontiguousarray(x[0]), st)["Y"]
        t = torch.from_numpy(np.ascontiguousarray(Y.view(np.float64)))
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([t.shape[0]]))
        mx = int(max(s.item() for s in sizes))
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype)
        pad[:t.shape[0]] = t
        parts = [torch.zeros_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad)
        if rank == 0:
            full = np.concatenate([parts[g][:int(sizes[g].item())].numpy() for g in range(world)], axis=0)
            gx = synth.datacube(gcfg)
            ref = oracle.run(oracle.OracleParams(cfg.C, cfg.T, gcfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), gx, st)["Y"]
            q.put(bool(np.array_equal(full.view(np.complex128), ref)))
    except Exception as e:  # surface worker errors in the parent
        if rank == 0:
            q.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["weak", "strong"])
def test_two_rank_doppler_shards_bitwise(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = q.get(timeout=10)
    assert res is True, res


def test_shard_rule_covers_everything():
    import synth
    for D in (1, 7, 8, 256, 1000):
        for G in (1, 2, 3, 4, 8):
            spans = [synth.shard_range(D, G, g) for g in range(G)]
            owned = [b for lo, c in spans for b in range(lo, lo + c)]
            assert owned == list(range(D))


def test_bench_inputs_match_global_cube():
    """bench.make_inputs at world 2: each rank's buffer is exactly the global weak cube's
    bins cube_bin0 .. +cube_bins (wrapped), and the owned slices tile the global bins."""
    import bench
    import synth
    cfg = synth.CONFIGS["tiny"].with_(T=3)
    full = None
    owned = []
    for r in range(2):
        gcfg, lo, cnt, b0, nb, x, st = bench.make_inputs(cfg, 2, r, cubes=1)
        if full is None:
            full = synth.datacube(gcfg)
        assert gcfg.D == 2 * cfg.D and cnt == cfg.D
        assert np.array_equal(x[0], full[(b0 + np.arange(nb)) % gcfg.D])
        owned += list(range(lo, lo + cnt))
    assert owned == list(range(2 * cfg.D))

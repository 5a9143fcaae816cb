"""Which (cube, tile, block) of the batched TC covariance are wrong / unwritten (dev check)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2203_06233_b200 as stap
cfg = synth.CONFIGS["small"]
M = 8
xs = np.stack([synth.datacube(cfg, i) for i in range(M)])
plan = stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), path="staged", batch=M)
p1 = stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), path="staged", batch=1)
out = torch.full(plan.cov_shape, float("nan"), dtype=torch.complex64, device="cuda")
plan.covariance(torch.from_numpy(xs).cuda().reshape(plan.cube_shape), out)
cb = out.cpu().numpy()
OB = 128 // cfg.C - cfg.T + 1
for n in range(M):
    c1 = p1.covariance(torch.from_numpy(xs[n:n+1]).cuda().reshape(p1.cube_shape)).cpu().numpy()[0]
    nanmask = np.isnan(cb[n]).any(axis=(-1, -2))          # [D][B]
    diff = ~np.isclose(cb[n], c1).all(axis=(-1, -2)) & ~nanmask
    print("cube", n, "unwritten (d,b)", int(nanmask.sum()), "wrong", int(diff.sum()), flush=True)
    if nanmask.any() or diff.any():
        bad = np.argwhere(nanmask | diff)
        tiles = sorted(set((int(d) // OB, int(b)) for d, b in bad))
        print("   tiles (td, b):", tiles[:20], len(tiles))
        # does the wrong value equal another cube's result?
        if diff.any():
            d, b = np.argwhere(diff)[0]
            for m in range(M):
                cm = p1.covariance(torch.from_numpy(xs[m:m+1]).cuda().reshape(p1.cube_shape)).cpu().numpy()[0]
                if np.allclose(cm[d, b], cb[n, d, b]): print("   (d,b)", d, b, "equals cube", m)

"""Repeat the tcgen05 covariance and report which (cube, bin, block, i, l) entries differ (dev check)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2203_06233_b200 as stap
cfg = synth.CONFIGS["large"].with_(D=int(sys.argv[1]) if len(sys.argv) > 1 else 32)
M = 2
x = np.stack([synth.datacube(cfg, i) for i in range(M)])
plan = stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), batch=M, path="staged")
dc = torch.from_numpy(x).cuda().reshape(plan.cube_shape)
c0 = plan.covariance(dc).cpu().numpy()
OB = 128 // cfg.C - cfg.T + 1
bad = {}
for rep in range(20):
    c = plan.covariance(dc).cpu().numpy()
    diff = c != c0
    if diff.any():
        idx = np.argwhere(diff)
        for n, d, b, i, l in idx[:2000]:
            key = (int(n), int(d) // OB, int(b))
            bad.setdefault(key, set()).add((int(d) % OB, int(i), int(l)))
print("tiles with differences (n, td, b):", sorted(bad)[:20], len(bad))
for k in sorted(bad)[:3]:
    ent = sorted(bad[k])
    print(k, "entries", len(ent), "sample (di, i, l):", ent[:12])
    print("   i set", sorted(set(e[1] for e in ent))[:20], " l set", sorted(set(e[2] for e in ent))[:20], " di set", sorted(set(e[0] for e in ent)))

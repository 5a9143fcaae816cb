"""TC covariance correctness vs SIMT over (C, T, D, K) variants -- dev check."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2203_06233_b200 as stap
cases = [("small", dict(), 8), ("small", dict(D=64), 4)]
for name, kw, M in cases:
    cfg = synth.CONFIGS[name].with_(**kw)
    plan = stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), path="staged", batch=M)
    x = torch.from_numpy(np.stack([synth.datacube(cfg, i) for i in range(M)])).cuda().reshape(plan.cube_shape)
    c1all = plan.covariance(x).cpu().numpy()
    os.environ["STAP_COV_SIMT"] = "1"
    plan2 = stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), path="staged", batch=M)
    del os.environ["STAP_COV_SIMT"]
    c2all = plan2.covariance(x).cpu().numpy()
    for n in range(M):
        c1, c2 = c1all[n], c2all[n]
        num = np.linalg.norm((c1 - c2).reshape(cfg.D, cfg.B, -1), axis=-1)
        den = np.linalg.norm(c2.reshape(cfg.D, cfg.B, -1), axis=-1)
        e = num / den
        print("  cube", n, "max", e.max(), "bad bins", np.where(e.max(axis=1) > 1e-4)[0][:10], "bad blocks", np.where(e.max(axis=0) > 1e-4)[0][:10])
    c1, c2 = c1all[M - 1], c2all[M - 1]
    num = np.linalg.norm((c1 - c2).reshape(cfg.D, cfg.B, -1), axis=-1)
    den = np.linalg.norm(c2.reshape(cfg.D, cfg.B, -1), axis=-1)
    e = num / den
    bad_d = np.where(e.max(axis=1) > 1e-4)[0]
    bad_b = np.where(e.max(axis=0) > 1e-4)[0]
    print(name, kw, "max", e.max(), "bad bins", bad_d[:12], len(bad_d), "bad blocks", bad_b[:8], len(bad_b), flush=True)
    if len(bad_d):
        d = bad_d[min(3, len(bad_d)-1)]; b = bad_b[0]
        print("   sample d", d, "b", b, "ratio diag tc/simt", np.round((np.diag(c1[d, b]).real / np.diag(c2[d, b]).real)[:8], 3))

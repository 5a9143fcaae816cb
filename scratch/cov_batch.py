"""Per-cube: batched covariance vs batch-1 covariance, for the TC and SIMT kernels (dev check)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2203_06233_b200 as stap
cfg = synth.CONFIGS["small"]
M = 8
xs = np.stack([synth.datacube(cfg, i) for i in range(M)])
for simt in (0, 1):
    if simt: os.environ["STAP_COV_SIMT"] = "1"
    plan = stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), path="staged", batch=M)
    p1 = stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), path="staged", batch=1)
    cb = plan.covariance(torch.from_numpy(xs).cuda().reshape(plan.cube_shape)).cpu().numpy()
    for n in range(M):
        c1 = p1.covariance(torch.from_numpy(xs[n:n+1]).cuda().reshape(p1.cube_shape)).cpu().numpy()[0]
        print("simt" if simt else "tc  ", "cube", n, "equal" if np.array_equal(cb[n], c1) else f"DIFF max {np.abs(cb[n]-c1).max():.3g}", flush=True)

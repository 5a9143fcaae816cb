"""Constant cubes (cube n = (n+1)(1+i)) through the batched TC covariance: which cube's rows did each tile read?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2203_06233_b200 as stap
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "small"]
M = int(sys.argv[2]) if len(sys.argv) > 2 else 8
xs = np.stack([np.full((cfg.D, cfg.C, cfg.R), (n + 1) * (1 + 1j), np.complex64) for n in range(M)])
plan = stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), path="staged", batch=M)
print(plan.description)
cb = plan.covariance(torch.from_numpy(xs).cuda().reshape(plan.cube_shape)).cpu().numpy()
for n in range(M):
    v = cb[n][:, :, 0, 1].real  # off-diagonal entry = 2 (n'+1)^2
    src = np.sqrt(v / 2) - 1
    bad = np.abs(src - n) > 1e-3
    print("cube", n, "bad entries", int(bad.sum()), "of", bad.size, "max src", float(src.max()), flush=True)
    if n == 1 and bad.any():
        dd = np.where(bad.any(axis=1))[0]
        print("   bad bins", dd.tolist())
        for d in dd[:40:4]:
            print("   d", d, "src per b", np.round(src[d], 2).tolist())

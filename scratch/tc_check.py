"""Compare the tcgen05 apply with the SIMT apply and the oracle (dev check)."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle
import paper_2203_06233_b200 as stap
for name in ("medium", "large"):
    cfg = synth.CONFIGS[name].with_(D=8)
    plan = stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam))
    print(name, plan.description, flush=True)
    x = synth.datacube(cfg)
    rng = np.random.default_rng(1)
    W = (rng.standard_normal((cfg.D, cfg.B, cfg.S, cfg.N)) + 1j * rng.standard_normal((cfg.D, cfg.B, cfg.S, cfg.N))).astype(np.complex64)
    dx = torch.from_numpy(x).cuda().reshape(plan.cube_shape)
    dw = torch.from_numpy(W).cuda().reshape(plan.weights_shape)
    y = plan.apply(dx, dw); torch.cuda.synchronize()
    Yr = oracle.apply(oracle.OracleParams(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), x, W)
    Y = y.cpu().numpy()[0]
    e = np.linalg.norm(Y - Yr, axis=-1) / np.linalg.norm(Yr, axis=-1)
    print(name, "tc vs oracle max rel-L2 per line", e.max(), "median", np.median(e), flush=True)

"""TC covariance vs the SIMT covariance (and timing) -- dev check."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2203_06233_b200 as stap
mode = sys.argv[1] if len(sys.argv) > 1 else "check"
for name in ("tiny", "small", "medium", "large"):
    cfg = synth.CONFIGS[name]
    if mode == "check" and name == "large":
        cfg = cfg.with_(D=48)
    M = {"tiny": 1, "small": 8, "medium": 4, "large": 1}[name] if mode == "check" else {"tiny": 1, "small": 64, "medium": 16, "large": 2}[name]
    plan = stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), batch=M, path="staged")
    x = torch.from_numpy(np.stack([synth.datacube(cfg, i % 4) for i in range(M)])).cuda().reshape(plan.cube_shape)
    if mode == "check":
        c1 = plan.covariance(x).cpu().numpy()
        os.environ["STAP_COV_SIMT"] = "1"
        plan2 = stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), batch=M, path="staged")
        del os.environ["STAP_COV_SIMT"]
        c2 = plan2.covariance(x).cpu().numpy()
        num = np.linalg.norm((c1 - c2).reshape(-1, cfg.N * cfg.N), axis=-1)
        den = np.linalg.norm(c2.reshape(-1, cfg.N * cfg.N), axis=-1)
        herm = np.array_equal(c1, np.conj(np.swapaxes(c1, -1, -2)))
        print(name, plan.description[:60], "max rel", (num / den).max(), "hermitian", herm, "nan", np.isnan(c1).any(), flush=True)
    else:
        for _ in range(3): plan.covariance(x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): plan.covariance(x)
        e1.record(); torch.cuda.synchronize()
        print(name, plan.description[:60], f"cov {e0.elapsed_time(e1)/10*1000:.1f} us/step (batch {M})", flush=True)

"""Small invocations of every entry point (fused and staged) for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2203_06233_b200 as stap
for name, D in (("tiny", 8), ("small", 16), ("medium", 8), ("large", 8)):
    cfg = synth.CONFIGS[name].with_(D=D) if name != "tiny" else synth.CONFIGS[name]
    plan = stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), batch=2)
    x = torch.from_numpy(np.stack([synth.datacube(cfg, i) for i in range(2)])).cuda()
    st = torch.from_numpy(synth.steering(cfg, "random")).cuda()
    y, info = plan.run(x, st)
    cov = plan.covariance(x)
    w, g, inf2 = plan.solve_weights(cov, st)
    y2 = plan.apply(x, w)
    torch.cuda.synchronize()
    print(name, plan.description, float((y - y2).abs().max()))

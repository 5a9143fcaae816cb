"""Time stap_run (fused) with a given library (env STAP_LIB) for configs on argv."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2203_06233_b200 as stap
for name in sys.argv[1:]:
    cfg = synth.CONFIGS[name]
    M = {"small": 64, "medium": 16}[name]
    plan = stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), batch=M)
    x = torch.from_numpy(np.stack([synth.datacube(cfg, i % 8) for i in range(M)])).cuda()
    st = torch.from_numpy(synth.steering(cfg)).cuda()
    for _ in range(3): plan.run(x, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): plan.run(x, st)
    e1.record(); torch.cuda.synchronize()
    print(os.path.basename(os.environ.get("STAP_LIB", "libstap.so")), name, f"{e0.elapsed_time(e1)/20:.3f} ms/step", plan.description)

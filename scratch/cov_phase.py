import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("STAP_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)), "libstap_covprof.so"))
import numpy as np, torch, synth
import paper_2203_06233_b200 as stap
name = sys.argv[1] if len(sys.argv) > 1 else "large"
cfg = synth.CONFIGS[name]
M = {"small": 64, "medium": 16, "large": 2}[name]
plan = stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), batch=M, path="staged")
x = torch.randn(plan.cube_shape + (2,), device="cuda").view(torch.complex64).reshape(plan.cube_shape)
plan.covariance(x); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)()
stap._lib.stap_debug_covtc_prof(buf)
v = list(buf); tiles = v[6]
print(name, "tiles(cta0-thread0 sum over CTAs)", tiles)
for i, nm in enumerate(["wait full", "wait mma_done(cc-2)", "main loop", "wait last mma", "band copy+delta", "R writes", "", "band copy only"]):
    if nm: print(f"  {nm:22s} {v[i] / tiles:10.0f} cycles/tile")

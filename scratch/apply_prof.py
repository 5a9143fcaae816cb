"""Run the staged apply of a config a few times (ncu target; dev only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2203_06233_b200 as stap
name = sys.argv[1] if len(sys.argv) > 1 else "large"
cfg = synth.CONFIGS[name]
plan = stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam))
print(plan.description, flush=True)
x = torch.randn(plan.cube_shape + (2,), device="cuda").view(torch.complex64).reshape(plan.cube_shape)
w = torch.randn(plan.weights_shape + (2,), device="cuda").view(torch.complex64).reshape(plan.weights_shape)
for _ in range(3):
    y = plan.apply(x, w)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    y = plan.apply(x, w)
e.record(); torch.cuda.synchronize()
print("apply ms", s.elapsed_time(e) / 10, flush=True)

import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2203_06233_b200 as stap
name = sys.argv[1] if len(sys.argv) > 1 else "large"
cfg = synth.CONFIGS[name]
M = {"small": 64, "medium": 16, "large": 2}[name]
plan = stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), batch=M, path="staged")
x = torch.randn(plan.cube_shape + (2,), device="cuda").view(torch.complex64).reshape(plan.cube_shape)
for _ in range(3): plan.covariance(x)
torch.cuda.synchronize()

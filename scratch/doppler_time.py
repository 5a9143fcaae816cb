"""Time stap_doppler per config (dev): HBM fraction of one read + one write of the cube."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2203_06233_b200 as stap
for name, M in (("small", 64), ("medium", 16), ("large", 2)):
    cfg = synth.CONFIGS[name]
    plan = stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), batch=M)
    raw = torch.randn(plan.cube_shape + (2,), device="cuda").view(torch.complex64).reshape(plan.cube_shape)
    w = torch.ones(cfg.D, device="cuda")
    out = torch.empty_like(raw)
    for _ in range(3):
        plan.doppler(raw, w, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        plan.doppler(raw, w, out)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10 / 1e3
    b = 2 * raw.numel() * 8
    print(name, M, f"{t * 1e6:.1f} us/step, {b / t / 1e9:.0f} GB/s, HBM frac {b / t / 6554e9:.3f}", flush=True)

"""Phase split of the fused kernel (profiling build scratch/libstap_prof.so)."""
import ctypes, os, sys
os.environ["STAP_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libstap_prof.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2203_06233_b200 as stap
lib = stap._lib
lib.stap_debug_fused_prof.argtypes = [ctypes.c_void_p]
for name in sys.argv[1:] or ["small"]:
    cfg = synth.CONFIGS[name]
    M = {"small": 16, "medium": 4, "large": 1, "tiny": 16}[name]
    plan = stap.StapPlan(stap.Dims(cfg.C, cfg.T, cfg.D, cfg.R, cfg.K, cfg.S, cfg.lam), batch=M)
    x = torch.from_numpy(np.stack([synth.datacube(cfg, i) for i in range(M)])).cuda()
    st = torch.from_numpy(synth.steering(cfg)).cuda()
    out = np.zeros(4, np.uint64)
    plan.run(x, st); torch.cuda.synchronize()
    lib.stap_debug_fused_prof(out.ctypes.data)
    plan.run(x, st); torch.cuda.synchronize()
    lib.stap_debug_fused_prof(out.ctypes.data)
    herk, solve, apply, tot = [int(v) for v in out]
    print(name, plan.description)
    print(f"  per-CTA cycles: total {tot:.3e}  herk {herk:.3e} ({herk/tot*100:.1f}%)")
    print(f"  per-segment sums: solve {solve:.3e} apply {apply:.3e}  (ratio solve/apply {solve/apply:.2f})")
    print(f"  segment-time share of CTA time: {(solve+apply)/tot:.2f} (segments per CTA {plan.description})")

"""c1 LogReg GD: fused cooperative run vs per-iteration steps (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1612_07448_b200 as fb
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(3)
s = torch.randn(100_000, 20, dtype=torch.float64, device=dev, generator=g)
r = torch.randn(10_000, 40, dtype=torch.float64, device=dev, generator=g)
k = torch.randint(1, 10_001, (100_000,), device=dev, generator=g)
nm = fb.build_pkfk(s, k, r)
y = torch.where(torch.randn(100_000, 1, dtype=torch.float64, device=dev, generator=g) >= 0, 1.0, -1.0)
for iters in (1, 20, 100):
    cfg = fb.TrainConfig(iterations=iters, step_size=1e-3)
    fb.logistic_gd(nm, y, cfg)
    ts = []
    for _ in range(5):
        ts.append(fb.logistic_gd(nm, y, cfg).wall_time_s)
    print(f"iters {iters:4d}: median wall {1e3 * float(np.median(ts)):.3f} ms", flush=True)
cfg = fb.TrainConfig(iterations=100, step_size=1e-9)
yl = torch.randn(100_000, 1, dtype=torch.float64, device=dev, generator=g)
fb.linreg_gd(nm, yl, cfg)
print(f"linreg iters 100: median wall {1e3 * float(np.median([fb.linreg_gd(nm, yl, cfg).wall_time_s for _ in range(5)])):.3f} ms")

"""c4 K-Means per-iteration time: median over 3 trials of (wall(21 iters) - wall(1 iter)) / 20.

usage: python tools/time_kmeans.py   (FB_KMEANS_FUSED=0 selects the unfused three-pass step)
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_07448_b200 as fb
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
n_s = 10_000_000
s = torch.randn(n_s, 20, dtype=torch.float64, device=dev, generator=g)
r1 = torch.randn(1_000_000, 40, dtype=torch.float64, device=dev, generator=g)
r2 = torch.randn(100_000, 60, dtype=torch.float64, device=dev, generator=g)
k1 = torch.randint(1, 1_000_001, (n_s,), device=dev, generator=g)
k2 = torch.randint(1, 100_001, (n_s,), device=dev, generator=g)
nm = fb.build_star(s, [(k1, r1), (k2, r2)])


def run(iters):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fb.kmeans(nm, fb.TrainConfig(iterations=iters, k=10))
    torch.cuda.synchronize()
    return time.perf_counter() - t0, out


run(2)
per = []
for _ in range(3):
    t1, _ = run(1)
    t21, out = run(21)
    per.append((t21 - t1) / 20)
per.sort()
print(f"FUSED={os.environ.get('FB_KMEANS_FUSED', '1')} ms_per_iter={per[1] * 1e3:.3f} "
      f"trace[-3:]={[f'{v:.12e}' for v in out.objective[-3:]]} "
      f"assign_sum={int(out.assignment.long().sum())}", flush=True)

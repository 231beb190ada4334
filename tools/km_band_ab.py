"""c4 K-Means: storage-order fused pass vs the FK-band layout, alternating in one process.

Per-iteration time = (wall(41 iters) - wall(1 iter)) / 40; prints the band build time too.
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_07448_b200 as fb
from paper_1612_07448_b200.normmat import NormalizedMatrix
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
n_s = 10_000_000
s = torch.randn(n_s, 20, dtype=torch.float64, device=dev, generator=g)
r1 = torch.randn(1_000_000, 40, dtype=torch.float64, device=dev, generator=g)
r2 = torch.randn(100_000, 60, dtype=torch.float64, device=dev, generator=g)
k1 = torch.randint(1, 1_000_001, (n_s,), device=dev, generator=g)
k2 = torch.randint(1, 100_001, (n_s,), device=dev, generator=g)
nm = fb.build_star(s, [(k1, r1), (k2, r2)])
nm.k if False else None
nm.indicator_blocks[0][0].sorted_order()  # warm the CUB sort kernels


def run(iters):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fb.kmeans(nm, fb.TrainConfig(iterations=iters, k=10))
    torch.cuda.synchronize()
    return time.perf_counter() - t0, out


default_min = NormalizedMatrix.BAND_KMEANS_MIN_BYTES
for mode in ("off", "on", "off", "on", "on"):
    NormalizedMatrix.BAND_KMEANS_MIN_BYTES = 0 if mode == "off" else default_min
    if mode == "on" and "band" not in nm._cache:
        torch.cuda.synchronize(); t0 = time.perf_counter()
        nm.kmeans_band_layout(10)
        torch.cuda.synchronize()
        print(f"band build {1e3 * (time.perf_counter() - t0):.2f} ms, bands={nm._cache['band'][0].n_bands}", flush=True)
    run(2)
    l0 = fb.launch_count()
    t1, _ = run(1)
    l1 = fb.launch_count()
    t41, out = run(41)
    print(f"band={mode} ms_per_iter={(t41 - t1) / 40 * 1e3:.3f} launches(1 iter)={l1 - l0} obj={out.objective[-1]:.12e} "
          f"assign_sum={int(out.assignment.long().sum())}", flush=True)

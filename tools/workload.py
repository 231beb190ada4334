"""Run one secondary workload a few times (for ncu / timing). usage: python tools/workload.py c3|c4|c5|c1 [reps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1612_07448_b200 as fb

which = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
if which == "c3":
    n_s, d_s, n_r, d_r = 10_000_000, 60, 500_000, 120
    s = torch.rand(n_s, d_s, dtype=torch.float64, device=dev, generator=g)
    r = torch.rand(n_r, d_r, dtype=torch.float64, device=dev, generator=g)
    key = torch.randint(1, n_r + 1, (n_s,), device=dev, generator=g)
    nm = fb.build_pkfk(s, key, r)
    from paper_1612_07448_b200.crossprod_impl import fk_sorted_order
    fk_sorted_order(nm.k)
    fn = lambda: fb.crossprod(nm)
elif which == "c4":
    n_s = 10_000_000
    s = torch.randn(n_s, 20, dtype=torch.float64, device=dev, generator=g)
    r1 = torch.randn(1_000_000, 40, dtype=torch.float64, device=dev, generator=g)
    r2 = torch.randn(100_000, 60, dtype=torch.float64, device=dev, generator=g)
    k1 = torch.randint(1, 1_000_001, (n_s,), device=dev, generator=g)
    k2 = torch.randint(1, 100_001, (n_s,), device=dev, generator=g)
    nm = fb.build_star(s, [(k1, r1), (k2, r2)])
    fn = lambda: fb.kmeans(nm, fb.TrainConfig(iterations=5, k=10))
elif which == "c5":
    import workloads as W
    gg = W.generate("c5")  # the seeded NumPy c5 inputs (Zipf(1.2) keys)
    (fk, r), = W.keys_1based(gg["parts"])
    nm = fb.build_pkfk(torch.from_numpy(gg["s"]).to(dev), torch.from_numpy(fk).to(dev), torch.from_numpy(r).to(dev))
    fn = lambda: fb.gnmf(nm, fb.TrainConfig(iterations=5, r=5))
else:
    rng = np.random.default_rng(1)
    nm = fb.build_pkfk(torch.from_numpy(rng.standard_normal((100_000, 20))).to(dev),
                       torch.from_numpy(rng.integers(1, 10_001, size=100_000)).to(dev),
                       torch.from_numpy(rng.standard_normal((10_000, 40))).to(dev))
    y = torch.where(torch.rand(100_000, 1, device=dev, dtype=torch.float64) > 0.5, 1.0, -1.0).double()
    fn = lambda: fb.logistic_gd(nm, y, fb.TrainConfig(iterations=20, step_size=1e-3))
torch.cuda.synchronize()
for i in range(reps):
    t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); print(which, "rep", i, "s", round(time.perf_counter() - t0, 5), flush=True)

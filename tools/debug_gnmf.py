import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1612_07448_b200 as fb
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
n_s, n_r = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000, 50_000
s = torch.rand(n_s, 10, dtype=torch.float64, device=dev, generator=g)
r = torch.rand(n_r, 40, dtype=torch.float64, device=dev, generator=g)
key = bench.zipf_keys_dev(n_s, n_r, 1.2, g, dev)
nm = fb.build_pkfk(s, key, r)
print("built", nm.r.shape, flush=True)
h = torch.rand(50, 5, dtype=torch.float64, device=dev)
print("lmm", fb.lmm(nm, h)[:1], flush=True)
res = fb.gnmf(nm, fb.TrainConfig(iterations=3, r=5, rng_seed=0))
print("gnmf", res.objective, flush=True)

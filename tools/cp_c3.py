"""c3 crossprod only (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_07448_b200 as fb
from paper_1612_07448_b200.crossprod_impl import fk_sorted_order
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
s = torch.rand(10_000_000, 60, dtype=torch.float64, device=dev, generator=g)
r = torch.rand(500_000, 120, dtype=torch.float64, device=dev, generator=g)
key = torch.randint(1, 500_001, (10_000_000,), device=dev, generator=g)
nm = fb.build_pkfk(s, key, r)
fk_sorted_order(nm.k)
for _ in range(int(os.environ.get("REPS", "3"))):
    fb.crossprod(nm)
torch.cuda.synchronize()

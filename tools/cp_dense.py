"""Dense S-only gram (10M x 60) for ncu captures (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_07448_b200 as fb
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
n, d = int(os.environ.get("N", 10_000_000)), int(os.environ.get("D", 60))
s = torch.rand(n, d, dtype=torch.float64, device=dev, generator=g)
nm = fb.as_normalized(s)
for _ in range(int(os.environ.get("REPS", "2"))):
    fb.crossprod(nm)
torch.cuda.synchronize()

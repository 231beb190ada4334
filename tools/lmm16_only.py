"""c2 LMM X100x16 only (for ncu captures of the S pass)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_07448_b200 as fb
g = torch.Generator(device="cuda").manual_seed(0)
n_r = int(os.environ.get("NR", "1000000"))
s = torch.randn(20_000_000, 20, dtype=torch.float64, device="cuda", generator=g)
r = torch.randn(n_r, 80, dtype=torch.float64, device="cuda", generator=g)
k = torch.randint(1, n_r + 1, (20_000_000,), device="cuda", generator=g)
nm = fb.build_pkfk(s, k, r)
x = torch.randn(100, int(os.environ.get("DX", "16")), dtype=torch.float64, device="cuda")
for _ in range(int(os.environ.get("REPS", "3"))):
    fb.lmm(nm, x)
torch.cuda.synchronize()

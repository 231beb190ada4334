"""Run one c2 operator a few times (for ncu launch lists). usage: python tools/c2_op.py lmm_x16|lmm_x1|rmm_x1|row_sums|col_sums [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_07448_b200 as fb
op = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = torch.Generator(device="cuda").manual_seed(0)
n_s, n_r = 20_000_000, 1_000_000
s = torch.randn(n_s, 20, dtype=torch.float64, device="cuda", generator=g)
r = torch.randn(n_r, 80, dtype=torch.float64, device="cuda", generator=g)
k = torch.randint(1, n_r + 1, (n_s,), device="cuda", generator=g)
nm = fb.build_pkfk(s, k, r)
x1 = torch.randn(100, 1, dtype=torch.float64, device="cuda")
x16 = torch.randn(100, 16, dtype=torch.float64, device="cuda")
xr = torch.randn(1, n_s, dtype=torch.float64, device="cuda")
fn = {"lmm_x16": lambda: fb.lmm(nm, x16), "lmm_x1": lambda: fb.lmm(nm, x1), "rmm_x1": lambda: fb.rmm(xr, nm),
      "row_sums": lambda: fb.row_sums(nm), "col_sums": lambda: fb.col_sums(nm)}[op]
torch.cuda.synchronize()
for _ in range(reps):
    fn()
torch.cuda.synchronize()

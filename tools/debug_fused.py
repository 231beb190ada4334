import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1612_07448_b200 as fb
from paper_1612_07448_b200.crossprod_impl import fk_sorted_order
dev = torch.device("cuda", 0)
for (n_s, d_s, n_r, d_r) in [(1000, 6, 50, 4), (5000, 20, 300, 8), (100000, 60, 5000, 40), (4, 2, 2, 2)]:
    g = torch.Generator(device=dev).manual_seed(1)
    s = torch.rand(n_s, d_s, dtype=torch.float64, device=dev, generator=g)
    r = torch.rand(n_r, d_r, dtype=torch.float64, device=dev, generator=g)
    key = torch.randint(1, n_r + 1, (n_s,), device=dev, generator=g)
    nm = fb.build_pkfk(s, key, r)
    fk_sorted_order(nm.k)
    os.environ["FB_CP_UNFUSED"] = "1"; a = fb.crossprod(nm)
    os.environ.pop("FB_CP_UNFUSED"); b = fb.crossprod(nm)
    torch.cuda.synchronize()
    ss = (a[:d_s, :d_s] - b[:d_s, :d_s]).abs().max().item()
    pp = (a[d_s:, :d_s] - b[d_s:, :d_s]).abs().max().item()
    rr = (a[d_s:, d_s:] - b[d_s:, d_s:]).abs().max().item()
    print(n_s, d_s, n_r, d_r, "SS", ss, "P", pp, "RR", rr, flush=True)
    if pp > 1e-9 and n_s <= 1000:
        ks = nm.k.target.long()
        B = torch.zeros(nm.k.cols, d_s, dtype=torch.float64, device=dev).index_add_(0, ks, s)
        print(" B rows", B[:3], flush=True)

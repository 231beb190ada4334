import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1612_07448_b200 as fb
from paper_1612_07448_b200.crossprod_impl import fk_sorted_order
dev = torch.device("cuda", 0)
for (n_s, d_s, n_r, d_r) in [(4, 2, 2, 2), (40, 2, 5, 2), (1000, 6, 50, 4)]:
    g = torch.Generator(device=dev).manual_seed(1)
    s = torch.rand(n_s, d_s, dtype=torch.float64, device=dev, generator=g)
    r = torch.rand(n_r, d_r, dtype=torch.float64, device=dev, generator=g)
    key = torch.randint(1, n_r + 1, (n_s,), device=dev, generator=g)
    nm = fb.build_pkfk(s, key, r)
    perm, fks = fk_sorted_order(nm.k)
    os.environ["FB_CP_DUMPB"] = "1"; o = fb.crossprod(nm); os.environ.pop("FB_CP_DUMPB")
    torch.cuda.synchronize()
    nb = min(o.numel(), nm.k.cols * d_s)
    got = o.flatten()[:nb].reshape(-1, d_s)
    ks = nm.k.target.long()
    B = torch.zeros(nm.k.cols, d_s, dtype=torch.float64, device=dev).index_add_(0, ks, s).flatten()[:nb].reshape(-1, d_s)
    print(n_s, d_s, "keys", nm.k.target[:8].tolist(), "perm", perm[:8].tolist(), "fks", fks[:8].tolist())
    print(" got", got[:4].tolist()); print(" ref", B[:4].tolist())
    print(" S", s[:4].tolist(), flush=True)

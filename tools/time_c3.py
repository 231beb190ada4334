"""c3 crossprod: fused vs unfused S pass (CUDA-event timing + agreement)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1612_07448_b200 as fb
from paper_1612_07448_b200.crossprod_impl import fk_sorted_order
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
n_s, d_s, n_r, d_r = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (10_000_000, 60, 500_000, 120)))
s = torch.rand(n_s, d_s, dtype=torch.float64, device=dev, generator=g)
r = torch.rand(n_r, d_r, dtype=torch.float64, device=dev, generator=g)
key = torch.randint(1, n_r + 1, (n_s,), device=dev, generator=g)
nm = fb.build_pkfk(s, key, r)
fk_sorted_order(nm.k)
res = {}
outs = {}
for mode in ("unfused", "fused"):
    if mode == "unfused":
        os.environ["FB_CP_UNFUSED"] = "1"
    else:
        os.environ.pop("FB_CP_UNFUSED", None)
    for _ in range(2):
        outs[mode] = fb.crossprod(nm)
    ts = []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fb.crossprod(nm); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    res[mode] = round(float(np.median(ts)), 4)
d = outs["fused"] - outs["unfused"]
res["rel_diff"] = float(d.norm() / outs["unfused"].norm())
res["sym"] = bool(torch.equal(outs["fused"], outs["fused"].t()))
print(res)

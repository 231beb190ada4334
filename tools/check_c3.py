"""c3-size crossprod vs a torch reference, fused and unfused, repeated (race hunting)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_07448_b200 as fb
from paper_1612_07448_b200.crossprod_impl import fk_sorted_order
dev = torch.device("cuda", 0)
n_s, d_s, n_r, d_r = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (10_000_000, 60, 500_000, 120)))
g = torch.Generator(device=dev).manual_seed(7)
s = torch.rand(n_s, d_s, dtype=torch.float64, device=dev, generator=g)
r = torch.rand(n_r, d_r, dtype=torch.float64, device=dev, generator=g)
key = torch.randint(1, n_r + 1, (n_s,), device=dev, generator=g)
nm = fb.build_pkfk(s, key, r)
fk_sorted_order(nm.k)
B = torch.zeros(nm.k.cols, d_s, dtype=torch.float64, device=dev).index_add_(0, nm.k.target.long(), s)
ref = torch.empty(d_s + d_r, d_s + d_r, dtype=torch.float64, device=dev)
ref[:d_s, :d_s] = s.t() @ s
ref[d_s:, :d_s] = nm.r.t() @ B
ref[:d_s, d_s:] = ref[d_s:, :d_s].t()
ref[d_s:, d_s:] = (nm.r * nm.k.counts[:, None]).t() @ nm.r
for mode in ("unfused", "fused"):
    if mode == "unfused":
        os.environ["FB_CP_UNFUSED"] = "1"
    else:
        os.environ.pop("FB_CP_UNFUSED", None)
    errs = []
    for _ in range(int(os.environ.get("REPS", "4"))):
        out = fb.crossprod(nm)
        torch.cuda.synchronize()
        errs.append(float((out - ref).norm() / ref.norm()))
    print(mode, ["%.1e" % e for e in errs], flush=True)

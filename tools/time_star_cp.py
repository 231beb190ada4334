"""Star-schema crossprod at the c4 shape (S 10M x 20, R1 1M x 40, R2 100k x 60): the fused composition
(per-part fused passes + pair-count cross blocks) vs the block-column path. CUDA events, median of 5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_07448_b200 as fb
from paper_1612_07448_b200 import crossprod_impl as CI
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
n_s = 10_000_000
d_s = int(os.environ.get("D_S", "20"))
s = torch.rand(n_s, d_s, dtype=torch.float64, device=dev, generator=g)
r1 = torch.rand(1_000_000, 40, dtype=torch.float64, device=dev, generator=g)
r2 = torch.rand(100_000, 60, dtype=torch.float64, device=dev, generator=g)
k1 = torch.randint(1, 1_000_001, (n_s,), device=dev, generator=g)
k2 = torch.randint(1, 100_001, (n_s,), device=dev, generator=g)
nm = fb.build_star(s, [(k1, r1), (k2, r2)])


def timed(fn):
    fn(); fn()
    ts = []
    for _ in range(5):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); out = fn(); e.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(e))
    return sorted(ts)[2], out


t_f, cp_f = timed(lambda: fb.crossprod(nm))
fused = CI._star_crossprod_fused
CI._star_crossprod_fused = CI._star_crossprod
t_b, cp_b = timed(lambda: fb.crossprod(nm))
CI._star_crossprod_fused = fused
dev_rel = float((cp_f - cp_b).abs().max() / cp_b.abs().max())
print(f"star crossprod c4 shape: fused composition {t_f:.2f} ms, block columns {t_b:.2f} ms, max rel diff {dev_rel:.2e}")

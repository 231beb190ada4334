"""c3 crossprod: whole-op time with the fused S pass's roles switched off one at a time
(FB_CP_DEBUG bit 0: walkers release only, bit 1: consumers issue no DMMA) and with ring overrides
(FB_CP_STAGES, FB_CP_FUSED_ROWS). Results of the debug modes are wrong by design: timing only."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1612_07448_b200 as fb
from paper_1612_07448_b200.crossprod_impl import fk_sorted_order
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
n_s, d_s, n_r, d_r = 10_000_000, 60, 500_000, 120
s = torch.rand(n_s, d_s, dtype=torch.float64, device=dev, generator=g)
r = torch.rand(n_r, d_r, dtype=torch.float64, device=dev, generator=g)
key = torch.randint(1, n_r + 1, (n_s,), device=dev, generator=g)
nm = fb.build_pkfk(s, key, r)
fk_sorted_order(nm.k)


def t(env):
    for k in ("FB_CP_DEBUG", "FB_CP_STAGES", "FB_CP_FUSED_ROWS", "FB_CP_NB2"):
        os.environ.pop(k, None)
    os.environ.update(env)
    for _ in range(2):
        fb.crossprod(nm)
    ts = []
    for _ in range(7):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fb.crossprod(nm); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print(env, round(float(np.median(ts)), 4), flush=True)


for env in ({}, {"FB_CP_NB2": "1"}, {"FB_CP_DEBUG": "1"}, {"FB_CP_DEBUG": "2"}, {"FB_CP_DEBUG": "3"}, {"FB_CP_STAGES": "3"},
            {"FB_CP_FUSED_ROWS": "32"}, {"FB_CP_FUSED_ROWS": "48"}, {"FB_CP_NB2": "1", "FB_CP_DEBUG": "1"}, {"FB_CP_FUSED_ROWS": "96"}, {"FB_CP_FUSED_ROWS": "128"}):
    try:
        t(env)
    except Exception as e:  # a ring configuration the kernel rejects
        print(env, "failed:", str(e)[:100], flush=True)

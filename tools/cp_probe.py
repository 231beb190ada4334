"""Crossprod timing probes (development aid): dense S-only gram vs the full factorized crossprod."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1612_07448_b200 as fb
from paper_1612_07448_b200.crossprod_impl import fk_sorted_order

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
s = torch.rand(10_000_000, 60, dtype=torch.float64, device=dev, generator=g)
dense = fb.as_normalized(s)
print("dense S gram ms", bench._events_ms(lambda: fb.crossprod(dense), 5))
r = torch.rand(500_000, 120, dtype=torch.float64, device=dev, generator=g)
key = torch.randint(1, 500_001, (10_000_000,), device=dev, generator=g)
nm = fb.build_pkfk(s, key, r)
fk_sorted_order(nm.k)
print("c3 crossprod ms", bench._events_ms(lambda: fb.crossprod(nm), 5))
# sorted-key copy of S: same gram, rows contiguous again (isolates the gather cost)
perm, _ = fk_sorted_order(nm.k)
s_sorted = s.index_select(0, perm.long())
print("dense sorted-S gram ms", bench._events_ms(lambda: fb.crossprod(fb.as_normalized(s_sorted)), 5))

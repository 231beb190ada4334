"""Split timings of the c2 LMM x16 / RMM passes (development aid, not the bench).

Prints the median CUDA-event time of: LMM x16 and RMM at c2; the same ops after the FK-sorted
order is built (RMM then runs its X·K as segmented sums); LMM x16 with a small R (z L2-resident,
isolates the S pass); LMM x16 with a small S (isolates the z-pass).
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1612_07448_b200 as fb  # noqa: E402


def timeit(fn, reps=10):
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return round(float(np.median(ts)), 4)


def make(n_s, d_s, n_r, d_r, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    s = torch.randn(n_s, d_s, dtype=torch.float64, device="cuda", generator=g)
    r = torch.randn(n_r, d_r, dtype=torch.float64, device="cuda", generator=g)
    k = torch.randint(1, n_r + 1, (n_s,), device="cuda", generator=g)
    return fb.build_pkfk(s, k, r)


res = {}
nm = make(20_000_000, 20, 1_000_000, 80)
d = 100
x16 = torch.randn(d, 16, dtype=torch.float64, device="cuda")
x8 = torch.randn(d, 8, dtype=torch.float64, device="cuda")
xr = torch.randn(1, 20_000_000, dtype=torch.float64, device="cuda")
res["lmm_x16"] = timeit(lambda: fb.lmm(nm, x16))
res["lmm_x8"] = timeit(lambda: fb.lmm(nm, x8))
res["rmm_x1"] = timeit(lambda: fb.rmm(xr, nm))
res["col_sums"] = timeit(lambda: fb.col_sums(nm))
nm.ensure_sorted()
nm._cache.pop("c_struct", None)
res["rmm_x1_sorted"] = timeit(lambda: fb.rmm(xr, nm))
res["lmm_x16_sorted_nm"] = timeit(lambda: fb.lmm(nm, x16))
del nm
torch.cuda.empty_cache()
nm = make(20_000_000, 20, 100_000, 80)
res["lmm_x16_nr100k"] = timeit(lambda: fb.lmm(nm, x16))
del nm
torch.cuda.empty_cache()
nm = make(20_000_000, 20, 500_000, 80)
res["lmm_x16_nr500k"] = timeit(lambda: fb.lmm(nm, x16))
del nm
torch.cuda.empty_cache()
nm = make(2_000_000, 20, 1_000_000, 80)
res["lmm_x16_ns2M"] = timeit(lambda: fb.lmm(nm, x16))
print(json.dumps(res, indent=1))

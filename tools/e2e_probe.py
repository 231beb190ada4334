"""Per-op timing of the c2 e2e path (public API, pinned host X, results to host) — development aid."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_07448_b200 as fb
g = torch.Generator(device="cuda").manual_seed(0)
n_s, d_s, n_r, d_r = 20_000_000, 20, 1_000_000, 80
s = torch.randn(n_s, d_s, dtype=torch.float64, device="cuda", generator=g)
r = torch.randn(n_r, d_r, dtype=torch.float64, device="cuda", generator=g)
k = torch.randint(1, n_r + 1, (n_s,), device="cuda", generator=g)
nm = fb.build_pkfk(s, k, r)
d = d_s + d_r
pin = lambda a: a.cpu().pin_memory()
hx1, hx16 = pin(torch.randn(d, 1, dtype=torch.float64)), pin(torch.randn(d, 16, dtype=torch.float64))
hxr = pin(torch.randn(1, n_s, dtype=torch.float64))
ops = {"lmm_x1": lambda: fb.lmm(nm, hx1), "lmm_x16": lambda: fb.lmm(nm, hx16), "rmm_x1": lambda: fb.rmm(hxr, nm),
       "row_sums": lambda: fb.row_sums(nm).cpu(), "col_sums": lambda: fb.col_sums(nm).cpu()}
for name, fn in ops.items():
    fn(); fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    print(f"{name:10s} {1e3 * (time.perf_counter() - t0) / 3:8.2f} ms", flush=True)

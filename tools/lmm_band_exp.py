"""c2 LMM X100x16 through an FK-band order (fb_normalized.band_*), CUDA events, median of 10.

env: BAND (bands, 0 = off), COPY (1: resident band-ordered S copy, 0: rows gathered via band_perm).
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1612_07448_b200 as fb
g = torch.Generator(device="cuda").manual_seed(0)
n_s, n_r, dx = 20_000_000, int(os.environ.get("NR", "1000000")), int(os.environ.get("DX", "16"))
s = torch.randn(n_s, 20, dtype=torch.float64, device="cuda", generator=g)
r = torch.randn(n_r, 80, dtype=torch.float64, device="cuda", generator=g)
k = torch.randint(1, n_r + 1, (n_s,), device="cuda", generator=g)
nm = fb.build_pkfk(s, k, r)
x = torch.randn(100, dx, dtype=torch.float64, device="cuda", generator=g)
ref = fb.lmm(nm, x).clone()
B = int(os.environ.get("BAND", "0"))
keep = []
if B:
    nm.c_struct()
    st = nm._cache["c_struct"]
    tgt = nm.indicator_blocks[0][0].target
    band = tgt.long() * B // n_r
    perm = torch.argsort(band, stable=True).to(torch.int32)
    bfk = tgt[perm.long()].contiguous()
    keep += [perm, bfk]
    st.band_perm = perm.data_ptr()
    st.band_fk[0] = bfk.data_ptr()
    if os.environ.get("COPY", "0") == "1":
        sb = s[perm.long()].contiguous()
        keep.append(sb)
        st.band_s = sb.data_ptr()
for _ in range(3):
    fb.lmm(nm, x)
ts = []
for _ in range(10):
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); out = fb.lmm(nm, x); e.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(e))
ts.sort()
nb = 8 * (n_s * 20 + n_r * 80) + 4 * n_s + 8 * (100 * dx + n_s * dx)
print(f"NR={n_r} DX={dx} BAND={B} COPY={os.environ.get('COPY', '0')} ms={ts[5]:.4f} GBps={nb / ts[5] / 1e6:.0f} "
      f"maxdiff={float((out - ref).abs().max()):.3g}", flush=True)

"""Small GNMF runs through the device path (debugging aid): uniform and Zipf keys."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
import paper_1612_07448_b200 as fb
n_s, n_r = int(os.environ.get("NS", "20000")), int(os.environ.get("NR", "500"))
rng = np.random.default_rng(0)
s = rng.random((n_s, 10)); r = rng.random((n_r, 40))
if os.environ.get("ZIPF", "0") == "1":
    key = W.zipf_keys(rng.random(n_s), W.zipf_cdf(n_r, 1.2)).astype(np.int64) + 1
else:
    key = rng.integers(1, n_r + 1, size=n_s)
nm = fb.build_pkfk(torch.from_numpy(s).cuda(), torch.from_numpy(key).cuda(), torch.from_numpy(r).cuda())
print("built", flush=True)
out = fb.gnmf(nm, fb.TrainConfig(iterations=int(os.environ.get("IT", "2")), r=5))
torch.cuda.synchronize()
print("ok", out.objective, flush=True)

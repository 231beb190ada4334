import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1612_07448_b200 as fb
for n, d in [(1000, 5), (1000, 12), (1000, 60), (7, 3)]:
    a = np.random.default_rng(0).random((n, d))
    cp = fb.crossprod(fb.as_normalized(a))
    ref = a.T @ a
    err = np.abs(cp - ref) / np.abs(ref).max()
    bad = np.argwhere(err > 1e-9)
    print(n, d, "maxerr", err.max(), "nbad", len(bad), bad[:6].tolist(), cp[0, :3], ref[0, :3], flush=True)

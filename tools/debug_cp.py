"""Crossprod smoke with synchronous launches (development aid): names the failing step."""
import os
import sys

os.environ.setdefault("CUDA_LAUNCH_BLOCKING", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np

import factorla_oracle as O
import paper_1612_07448_b200 as fb

for (n_s, d_s, n_r, d_r) in [(3, 2, 2, 2), (400, 12, 25, 18), (300_001, 60, 15_000, 120)]:
    rng = np.random.default_rng(0)
    s = rng.random((n_s, d_s))
    r = rng.random((n_r, d_r))
    key = rng.integers(1, n_r + 1, size=n_s)
    nm = fb.build_pkfk(s, key, r)
    try:
        cp = fb.crossprod(nm)
        print(n_s, d_s, n_r, d_r, "dev", O.max_rel_deviation(cp, O.crossprod(O.build_pkfk(s, key, r))), flush=True)
    except Exception as e:  # noqa: BLE001
        print(n_s, d_s, n_r, d_r, "FAILED", repr(e), flush=True)
        break

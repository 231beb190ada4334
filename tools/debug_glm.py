import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1612_07448_b200 as fb
for n_s in (3, 100, 5000):
    rng = np.random.default_rng(0)
    s = rng.random((n_s, 2)); r = rng.random((2, 2)); key = rng.integers(1, 3, size=n_s)
    nm = fb.build_pkfk(s, key, r)
    print("lmm", n_s, fb.lmm(nm, np.ones((4, 1)))[:2].ravel(), flush=True)
    y = np.where(rng.random((n_s, 1)) > 0.5, 1.0, -1.0)
    out = fb.logistic_gd(nm, y, fb.TrainConfig(iterations=2, step_size=1e-3))
    print("glm", n_s, out.weights.ravel(), flush=True)

import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import factorla_oracle as O
import paper_1612_07448_b200 as fb
n_s, d_s, shapes, seed = (40_001, 1, [(97, 5), (1000, 2)], 3)
rng = np.random.default_rng(seed)
s = rng.standard_normal((n_s, d_s))
parts = [(rng.integers(1, n_r + 1, size=n_s), rng.standard_normal((n_r, d_r))) for n_r, d_r in shapes]
ref = O.build_star(s, parts)
nm = fb.build_star(s, parts)
rng = np.random.default_rng(seed + 100)
n, d = ref.shape
for m in (1, 3, 10, 17):
    p = rng.standard_normal((n, m))
    a = fb.lmm(nm.T, p); b = O.lmm(ref.T, p)
    print("tmm", m, O.max_rel_deviation(a, b), np.abs(a - b).max(axis=1))
    a = fb.rmm(p.T.copy(), nm); b = O.rmm(p.T, ref)
    print("rmm", m, O.max_rel_deviation(a, b), np.abs(a - b).max(axis=0))
print("col_sums", O.max_rel_deviation(fb.col_sums(nm), O.col_sums(ref)))

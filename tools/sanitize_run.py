"""Small-shape pass over every ring kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck). usage: compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__)))]
import numpy as np
import torch

import paper_1612_07448_b200 as fb

rng = np.random.default_rng(5)
n, n_r = 20_011, 1_003
s = rng.standard_normal((n, 20))
r = rng.standard_normal((n_r, 40))
k = rng.integers(1, n_r + 1, size=n)
nm = fb.build_pkfk(s, k, r)
for dx in (1, 3, 10, 16):
    fb.lmm(nm, rng.standard_normal((60, dx)))              # rowdot / DMMA S pass + z pass
fb.lmm(nm.T, rng.standard_normal((n, 3)))                 # colreduce + gatherer-warp REDs
fb.rmm(rng.standard_normal((2, n)), nm)
fb.row_sums(nm); fb.col_sums(nm); fb.sum_all(nm)
fb.crossprod(nm)                                          # fused FK-sorted S pass + walkers + carry fixup
y = np.where(rng.standard_normal((n, 1)) > 0, 1.0, -1.0)
fb.logistic_gd(nm, y, fb.TrainConfig(iterations=2, step_size=1e-3))   # cooperative glm_run
fb.kmeans(nm, fb.TrainConfig(iterations=2, k=5))                      # assign + onehot + histograms
zk = np.minimum((rng.zipf(1.3, size=n) - 1), n_r - 1) + 1             # skewed keys: segsum + hot bins
nz = fb.build_pkfk(np.abs(s[:, :6]), zk, np.abs(r[:, :5]))
fb.gnmf(nz, fb.TrainConfig(iterations=2, r=3))
fb.lmm(nz.T, rng.standard_normal((n, 2)))
st = fb.build_star(s, [(k, r), (rng.integers(1, 51, size=n), rng.standard_normal((50, 6)))])
fb.crossprod(st); fb.kmeans(st, fb.TrainConfig(iterations=2, k=4))
torch.cuda.synchronize()
print("sanitize pass ok, launches", fb.launch_count())

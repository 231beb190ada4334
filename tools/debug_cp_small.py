import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1612_07448_b200 as fb
rng = np.random.default_rng(0)
s = rng.random((400, 12)); r = rng.random((25, 18)); key = rng.integers(1, 26, size=400)
nm = fb.build_pkfk(s, key, r)
print(fb.crossprod(nm)[0, :3])

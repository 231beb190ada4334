"""Run every wide fixture of tests/test_fuzz_gpu.py and list the distinct failures."""
import os, sys, traceback, warnings
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (root, os.path.join(root, "oracle"), os.path.join(root, "tests")):
    sys.path.insert(0, p)
import numpy as np
import test_fuzz_gpu as F
import paper_1612_07448_b200 as fb
warnings.simplefilter("ignore")
n = int(sys.argv[1]) if len(sys.argv) > 1 else F.N_WIDE
bad = 0
for seed in range(n):
    try:
        F._one_wide_fixture(fb, 130_000 + seed)
    except Exception as e:
        bad += 1
        rng = np.random.default_rng(130_000 + seed)
        q = int(rng.integers(1, 3)); nn = int(rng.integers(500, 20_000)); ds = int(rng.integers(60, 301))
        tb = traceback.extract_tb(e.__traceback__)
        where = [(os.path.basename(f.filename), f.lineno) for f in tb][-2:]
        print(f"seed {130_000 + seed} q={q} n={nn} d_s={ds}: {type(e).__name__}: {str(e)[:120]} at {where}", flush=True)
print("failures", bad, "of", n)

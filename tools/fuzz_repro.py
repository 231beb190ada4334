"""Replay one fixture of tests/test_fuzz_gpu.py by seed, operator by operator (usage: fuzz_repro.py SEED)."""
import os, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (root, os.path.join(root, "oracle"), os.path.join(root, "tests")):
    sys.path.insert(0, p)
import numpy as np
import factorla_oracle as O
import test_fuzz_gpu as F
import paper_1612_07448_b200 as fb

seed = int(sys.argv[1])
kind, rng, data = F._draw(seed)
nm, ref = F._build(fb, kind, data)
t = O.materialize(ref)
n, d = t.shape
print(kind, "T", t.shape, "blocks", [(None if e is None else e.cols, tuple(f.shape)) for e, f in nm.blocks])
for dx in (1, 2, 3, 4, 5, 7, 8, 9, 12, 16, 17, 19):
    x = np.random.default_rng(dx).standard_normal((d, dx))
    got = F._np(fb.lmm(nm, x))
    want = O.lmm(ref, x)
    dev = O.max_rel_deviation(got, want)
    bad_cols = np.nonzero(np.abs(got - want).max(axis=0) > 1e-9 * np.abs(want).max())[0]
    bad_rows = np.nonzero(np.abs(got - want).max(axis=1) > 1e-9 * np.abs(want).max())[0]
    print(f"lmm dx={dx}: dev {dev:.2e} bad cols {bad_cols.tolist()[:20]} bad rows {len(bad_rows)} first {bad_rows[:8].tolist()}")

"""Rowdot LMM (d_x = 1) on small star shapes around a failing fuzz fixture."""
import os, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (root, os.path.join(root, "oracle")):
    sys.path.insert(0, p)
import numpy as np
import factorla_oracle as O
import paper_1612_07448_b200 as fb

def run(n, d_s, shapes, keymode, dx=1):
    rng = np.random.default_rng(1)
    s = rng.standard_normal((n, d_s))
    parts = []
    for (n_r, d_r), km in zip(shapes, keymode):
        key = np.full(n, min(9, n_r)) if km == "one" else rng.integers(1, n_r + 1, size=n)
        parts.append((key, rng.standard_normal((n_r, d_r))))
    nm = fb.build_star(s, parts) if len(parts) > 1 else fb.build_pkfk(s, *parts[0])
    ref = O.build_star(s, parts)
    x = rng.standard_normal((d_s + sum(d for _, d in shapes), dx))
    got = fb.lmm(nm, x); got = got.cpu().numpy() if hasattr(got, "cpu") else got
    want = O.lmm(ref, x)
    bad = np.nonzero(np.abs(got - want).max(axis=1) > 1e-9 * np.abs(want).max())[0]
    print(f"n={n} d_s={d_s} parts={shapes} keys={keymode} dx={dx}: dev {O.max_rel_deviation(got, want):.1e} bad rows {len(bad)} {bad[:6].tolist()}", flush=True)

for n_r in (8, 64, 100, 128, 129, 152, 1000, 5000):
    run(2419, 20, [(n_r, 16)], ["u"])
for d_r in (8, 15, 17, 24, 32, 40):
    run(2419, 20, [(152, d_r)], ["u"])
for n in (31, 32, 33, 255, 257, 1024, 5000, 40000):
    run(n, 20, [(152, 16)], ["u"])
run(2419, 20, [(152, 16)], ["u"], dx=2)
run(2419, 20, [(152, 16)], ["u"], dx=4)

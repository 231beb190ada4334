"""Run every driver fixture of tests/test_fuzz_gpu.py and list the failures (no stop at the first)."""
import os, sys, warnings
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (root, os.path.join(root, "oracle"), os.path.join(root, "tests")):
    sys.path.insert(0, p)
import test_fuzz_gpu as F
import paper_1612_07448_b200 as fb
warnings.simplefilter("ignore")
n = int(sys.argv[1]) if len(sys.argv) > 1 else F.N_DRIVER
bad = 0
for seed in range(n):
    try:
        F._one_driver_fixture(fb, 50_000 + seed)
    except Exception as e:
        bad += 1
        kind, rng, data = F._draw(50_000 + seed)
        shape = kind if kind in ("mn", "multimn") else (data[0].shape, [(k.shape[0], r.shape) for k, r in data[1]])
        print(f"seed {50_000 + seed} {kind} {shape}: {type(e).__name__}: {str(e)[:160]}", flush=True)
print("failures", bad, "of", n)

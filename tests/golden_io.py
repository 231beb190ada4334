"""Load the committed golden fixtures (tests/golden/*.npz, made by oracle/gen_golden.py)."""
import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _all():
    return sorted(os.path.splitext(os.path.basename(p))[0] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def names():
    """PK-FK / star fixtures (S plus keyed attribute tables)."""
    return [n for n in _all() if not n.startswith(("mn_", "multimn_")) and n != "products"]


def mn_names():
    """M:N and multi-table M:N fixtures (normmat.py:240-319)."""
    return [n for n in _all() if n.startswith(("mn_", "multimn_"))]


def load(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def parts(g):
    return [(g[f"key{i}"], g[f"r{i}"]) for i in range(int(g["q"]))]

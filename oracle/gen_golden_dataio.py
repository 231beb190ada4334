"""Golden datasets for the ingestion path, made by the LIVE reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden_dataio.py

For each case it writes a dataset directory ``tests/golden/dataio/<case>/`` — by the
reference's own generators (``dataio.gen_pkfk`` / ``gen_mn``, dataio.py:407-457) or, for the
string-keyed star schema, by hand through its ``write_dense_csv`` / ``write_triplet`` — then
loads it with the reference's ``dataio.load`` (dataio.py:256-322) and stores the materialized
T (``normmat.materialize``, normmat.py:138), the target and the shape as
``tests/golden/dataio/<case>.npz``. Tests compare the device loader with these and the
repo's generators with the committed files byte for byte. The GPU box never reads
/root/reference.
"""

import json
import os
import shutil
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "dataio")


def _star_strings(dataio, out):
    """Two attribute tables: one keyed by string ids (pk column), one positional triplet."""
    rng = np.random.default_rng(7)
    os.makedirs(out, exist_ok=True)
    n_s, ids = 23, ["u07", "u03", "x9", "u11", "a0", "zz"]  # "zz" never referenced: dropped
    keys_a = rng.choice(ids[:5], size=n_s)
    keys_b = rng.integers(1, 5, size=n_s)
    keys_b[:4] = np.arange(1, 5)
    s = rng.random((n_s, 3))
    y = rng.random(n_s)
    with open(os.path.join(out, "entity.csv"), "w") as fh:
        fh.write("y,ka,f0,kb,f1,f2\n")
        for i in range(n_s):
            fh.write(f"{y[i]:.17g},{keys_a[i]},{s[i, 0]:.17g},{keys_b[i]},{s[i, 1]:.17g},{s[i, 2]:.17g}\n")
    ra = rng.standard_normal((len(ids), 2))
    with open(os.path.join(out, "ta.csv"), "w") as fh:
        fh.write("f0,name,f1\n")
        for i, name in enumerate(ids):
            fh.write(f"{ra[i, 0]:.17g},{name},{ra[i, 1]:.17g}\n")
    rb = np.zeros((4, 30))
    rb[0, 3], rb[1, 29], rb[2, 0], rb[3, 17], rb[3, 18] = 1.5, -2.0, 0.25, 3.0, 4.0
    dataio.write_triplet(os.path.join(out, "tb.triplet"), rb)
    schema = {
        "entity": {"path": "entity.csv", "target": "y",
                   "keys": [{"column": "ka", "table": "A", "kind": "pkfk"},
                            {"column": "kb", "table": "B", "kind": "pkfk"}]},
        "tables": [{"id": "A", "path": "ta.csv", "pk": "name"}, {"id": "B", "path": "tb.triplet", "pk": None}],
    }
    with open(os.path.join(out, "schema.json"), "w") as fh:
        json.dump(schema, fh, indent=2, sort_keys=True)
        fh.write("\n")
    return os.path.join(out, "schema.json")


def main():
    sys.path.insert(0, REF)
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    from factorla import dataio, kernel, normmat

    if os.path.isdir(OUT):
        shutil.rmtree(OUT)
    os.makedirs(OUT)
    cases = {
        "pkfk_dense": lambda d: dataio.gen_pkfk(dataio.SynthParams(n_s=40, n_r=8, d_s=3, d_r=4, seed=3), d),
        # density 3%: the attribute table is written as a triplet, both tables load as CSR
        "pkfk_sparse": lambda d: dataio.gen_pkfk(
            dataio.SynthParams(n_s=60, n_r=10, d_s=40, d_r=30, density=0.03, seed=5), d),
        "mn": lambda d: dataio.gen_mn(dataio.SynthParams(n_s=30, n_r=12, d_s=2, d_r=3, n_u=5, seed=9), d),
        "star_strings": lambda d: _star_strings(dataio, d),
    }
    for name, make in cases.items():
        d = os.path.join(OUT, name)
        schema = make(d)
        nm, y = dataio.load(schema)
        t = kernel.to_dense(normmat.materialize(nm))
        meta = {"variant": nm.variant, "sparse_s": int(kernel.is_sparse(nm.blocks[0][1]) if hasattr(kernel, "is_sparse")
                                                          else hasattr(nm.blocks[0][1], "tocsr"))}
        np.savez(os.path.join(OUT, name + ".npz"), t=t, y=np.zeros((0, 1)) if y is None else np.asarray(y),
                 shape=np.array(t.shape), variant=np.array(nm.variant), sparse_s=np.array(meta["sparse_s"]))
        print(name, t.shape, nm.variant, "sparse S" if meta["sparse_s"] else "dense S")


if __name__ == "__main__":
    main()

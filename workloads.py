"""Seeded synthetic inputs for the BASELINE.json configurations.

Bench / test infrastructure, not product code. Every configuration is drawn on the host
with NumPy ``default_rng``: the row-independent arrays (R tables, X operands, model
truth) from ``default_rng([seed, 0])``, and the row-indexed arrays (S rows, FK targets,
per-row operands, noise) in blocks of ``BLOCK`` rows, block b from
``default_rng([seed, b + 1])``. Any row range therefore has the same bytes whether it is
drawn alone (a rank's shard of a strong-scaling run) or as part of the whole matrix (the
parity tests, the CPU reference), and the blocks are drawn on parallel threads.

Conventions:
* N(0,1) = ``standard_normal``, U[0,1) = ``random``;
* FK targets are int32, 0-based, uniform over the R rows unless stated; the builders take
  1-based keys (``keys_1based``: fk + 1, normmat.py:182-198);
* Zipf(s) keys: inverse CDF of p(k) ∝ k^-s over the R rows (``zipf_keys``);
* c3's noise is N(0, 0.01²) (σ = 0.01; BASELINE.json leaves σ vs σ² open).

The paper's real datasets are not used (not in this container); these shapes and value
distributions are BASELINE.json's ``configs``.
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

SEEDS = {"c1": 101, "c2": 102, "c3": 103, "c4": 104, "c5": 105}
BLOCK = 500_000

SHAPES = {
    "c1": dict(n_s=100_000, d_s=20, parts=[(10_000, 40)], dist="normal"),
    "c2": dict(n_s=20_000_000, d_s=20, parts=[(1_000_000, 80)], dist="normal"),
    "c3": dict(n_s=10_000_000, d_s=60, parts=[(500_000, 120)], dist="uniform"),
    "c4": dict(n_s=10_000_000, d_s=20, parts=[(1_000_000, 40), (100_000, 60)], dist="normal"),
    "c5": dict(n_s=5_000_000, d_s=10, parts=[(50_000, 40)], dist="uniform"),
}


def zipf_cdf(n_r, s):
    p = np.arange(1, n_r + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(p)
    cdf /= cdf[-1]
    return cdf


def zipf_keys(u, cdf):
    """0-based int32 targets from U[0,1) draws u by the inverse CDF (P(k) ∝ (k+1)^-s)."""
    return np.minimum(np.searchsorted(cdf, u, side="right"), cdf.size - 1).astype(np.int32)


def _fill(rng, dist, out):
    if dist == "normal":
        rng.standard_normal(out=out)
    else:
        rng.random(out=out)


def _shared(name):
    """Row-independent arrays of a config, drawn from default_rng([seed, 0])."""
    sh = SHAPES[name]
    rng = np.random.default_rng([SEEDS[name], 0])
    rs = []
    for n_r, d_r in sh["parts"]:
        r = np.empty((n_r, d_r))
        _fill(rng, sh["dist"], r)
        rs.append(r)
    d = sh["d_s"] + sum(d_r for _, d_r in sh["parts"])
    extra = {}
    if name == "c1":
        extra["x"] = rng.standard_normal((d, 1))
        extra["w_true"] = rng.standard_normal((d, 1))
    elif name == "c2":
        extra["x1"] = rng.standard_normal((d, 1))
        extra["x16"] = rng.standard_normal((d, 16))
    elif name == "c3":
        extra["w_true"] = rng.standard_normal((d, 1))
    return rs, extra


def _rows(name, lo, hi, rs, extra):
    """Row-indexed arrays for rows [lo, hi), drawn block by block on parallel threads."""
    sh = SHAPES[name]
    n = hi - lo
    d_s = sh["d_s"]
    s = np.empty((n, d_s))
    fks = [np.empty(n, dtype=np.int32) for _ in rs]
    xr = np.empty((1, n)) if name == "c2" else None
    noise = np.empty((n, 1)) if name == "c3" else None
    cdf = zipf_cdf(rs[0].shape[0], 1.2) if name == "c5" else None

    def block(b):
        b0, b1 = b * BLOCK, min((b + 1) * BLOCK, sh["n_s"])
        rng = np.random.default_rng([SEEDS[name], b + 1])
        bs = np.empty((b1 - b0, d_s))
        _fill(rng, sh["dist"], bs)
        bfk = []
        for r in rs:
            if cdf is not None:
                bfk.append(zipf_keys(rng.random(b1 - b0), cdf))
            else:
                bfk.append(rng.integers(0, r.shape[0], size=b1 - b0, dtype=np.int32))
        bx = rng.standard_normal(b1 - b0) if xr is not None else None
        bn = rng.standard_normal(b1 - b0) if noise is not None else None
        c0, c1 = max(lo, b0), min(hi, b1)  # overlap with the requested range
        s[c0 - lo:c1 - lo] = bs[c0 - b0:c1 - b0]
        for f, bf in zip(fks, bfk):
            f[c0 - lo:c1 - lo] = bf[c0 - b0:c1 - b0]
        if bx is not None:
            xr[0, c0 - lo:c1 - lo] = bx[c0 - b0:c1 - b0]
        if bn is not None:
            noise[c0 - lo:c1 - lo, 0] = bn[c0 - b0:c1 - b0]

    blocks = range(lo // BLOCK, (hi - 1) // BLOCK + 1) if n > 0 else range(0)
    with ThreadPoolExecutor(max_workers=max(1, min(16, os.cpu_count() or 1))) as ex:
        list(ex.map(block, blocks))
    return s, fks, xr, noise


def _t_times(s, parts, w):
    """T·w on the host without materialising T (labels / targets only)."""
    d_s = s.shape[1]
    out = s @ w[:d_s]
    off = d_s
    for fk, r in parts:
        out += (r @ w[off:off + r.shape[1]])[fk]
        off += r.shape[1]
    return out


def generate(name, lo=0, hi=None):
    """Inputs of config ``name`` for entity rows [lo, hi) (default: all) as host arrays.

    Keys: ``s`` (rows × d_S f64), ``parts`` = [(fk int32 0-based, R f64)] (R whole), ``n_s``
    (the config's full row count), ``lo``/``hi``, and the config's operands / driver settings.
    """
    sh = SHAPES[name]
    hi = sh["n_s"] if hi is None else hi
    rs, extra = _shared(name)
    s, fks, xr, noise = _rows(name, lo, hi, rs, extra)
    parts = list(zip(fks, rs))
    out = {"name": name, "seed": SEEDS[name], "n_s": sh["n_s"], "lo": lo, "hi": hi, "s": s, "parts": parts}
    out.update(extra)
    if name == "c1":
        out["y"] = np.where(_t_times(s, parts, extra["w_true"]) >= 0, 1.0, -1.0)  # ties -> +1
        out.update(iterations=20, step=1e-3)
    elif name == "c2":
        out["xr"] = xr
    elif name == "c3":
        out["y"] = _t_times(s, parts, extra["w_true"]) + 0.01 * noise
    elif name == "c4":
        out.update(k=10, iterations=20, kmeans_seed=0)
    elif name == "c5":
        out.update(r=5, iterations=20, gnmf_seed=0)
    return out


def keys_1based(parts):
    """[(key int64 1-based, R)] for build_pkfk / build_star."""
    return [(fk.astype(np.int64) + 1, r) for fk, r in parts]


def algorithmic_bytes_c2(n_s, d_s, n_r, d_r):
    """Per-operator algorithmic bytes of the c2 suite (inputs + outputs once)."""
    d = d_s + d_r
    fac = 8 * (n_s * d_s + n_r * d_r)
    fk = 4 * n_s
    return {
        "lmm_x1": fac + fk + 8 * (d + n_s),
        "lmm_x16": fac + fk + 8 * (16 * d + 16 * n_s),
        "rmm_x1": fac + fk + 8 * (n_s + d),
        "row_sums": fac + fk + 8 * n_s,
        "col_sums": fac + 8 * (n_r + d),  # cached counts (indicator.py:61-66) replace the FK read
    }

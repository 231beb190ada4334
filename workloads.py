"""Seeded synthetic inputs for the BASELINE.json configurations.

Bench / test infrastructure, not product code: every configuration is drawn on the host
by a NumPy ``default_rng(seed)`` (one seed per config, ``SEEDS``), in the draw order
written below, so the GPU path, the reference (stock ``factorla``) and the CPU oracle
all see the same bytes. Conventions:

* N(0,1) = ``standard_normal``, U[0,1) = ``random``;
* FK targets are int32, 0-based, uniform (``integers(0, n_R)``) unless stated; the
  builders take 1-based keys (``fk + 1``, normmat.py:182-198);
* Zipf(s) keys: inverse CDF of p(k) ∝ k^-s over the R rows (``zipf_keys``);
* c3's noise is N(0, 0.01²) (σ = 0.01 — BASELINE.json leaves σ vs σ² open; recorded
  here and in DESIGN.md).

The paper's real datasets are not used (not in this container); these shapes and value
distributions are BASELINE.json's ``configs``.
"""
import numpy as np

SEEDS = {"c1": 101, "c2": 102, "c3": 103, "c4": 104, "c5": 105}

SHAPES = {
    "c1": dict(n_s=100_000, d_s=20, parts=[(10_000, 40)]),
    "c2": dict(n_s=20_000_000, d_s=20, parts=[(1_000_000, 80)]),
    "c3": dict(n_s=10_000_000, d_s=60, parts=[(500_000, 120)]),
    "c4": dict(n_s=10_000_000, d_s=20, parts=[(1_000_000, 40), (100_000, 60)]),
    "c5": dict(n_s=5_000_000, d_s=10, parts=[(50_000, 40)]),
}


def zipf_keys(rng, n, n_r, s):
    """0-based int32 targets with P(k) ∝ (k+1)^-s: inverse CDF of one U[0,1) draw per row."""
    p = np.arange(1, n_r + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(p)
    cdf /= cdf[-1]
    u = rng.random(n)
    return np.minimum(np.searchsorted(cdf, u, side="right"), n_r - 1).astype(np.int32)


def _t_times(s, parts, w):
    """T·w on the host without materialising T (labels / targets only)."""
    d_s = s.shape[1]
    out = s @ w[:d_s]
    off = d_s
    for fk, r in parts:
        out += (r @ w[off:off + r.shape[1]])[fk]
        off += r.shape[1]
    return out


def generate(name, scale=1.0):
    """Inputs of config ``name`` as a dict of host arrays.

    Keys: ``s`` (n_S × d_S f64), ``parts`` = [(fk int32 0-based, R f64)], plus the
    config's operands. ``scale`` < 1 shrinks every row count (tests of the generator
    itself); parity runs use 1.0.
    """
    rng = np.random.default_rng(SEEDS[name])
    sh = SHAPES[name]
    n_s = max(1, int(sh["n_s"] * scale))
    d_s = sh["d_s"]
    dims = [(max(1, int(n_r * scale)), d_r) for n_r, d_r in sh["parts"]]
    out = {"name": name, "seed": SEEDS[name]}
    if name == "c1":
        s = rng.standard_normal((n_s, d_s))
        (n_r, d_r), = dims
        r = rng.standard_normal((n_r, d_r))
        fk = rng.integers(0, n_r, size=n_s, dtype=np.int32)
        d = d_s + d_r
        out["x"] = rng.standard_normal((d, 1))
        w_true = rng.standard_normal((d, 1))
        tw = _t_times(s, [(fk, r)], w_true)
        out["y"] = np.where(tw >= 0, 1.0, -1.0)  # ties -> +1
        out.update(s=s, parts=[(fk, r)], iterations=20, step=1e-3)
    elif name == "c2":
        s = rng.standard_normal((n_s, d_s))
        (n_r, d_r), = dims
        r = rng.standard_normal((n_r, d_r))
        fk = rng.integers(0, n_r, size=n_s, dtype=np.int32)
        d = d_s + d_r
        out["x1"] = rng.standard_normal((d, 1))
        out["x16"] = rng.standard_normal((d, 16))
        out["xr"] = rng.standard_normal((1, n_s))
        out.update(s=s, parts=[(fk, r)])
    elif name == "c3":
        s = rng.random((n_s, d_s))
        (n_r, d_r), = dims
        r = rng.random((n_r, d_r))
        fk = rng.integers(0, n_r, size=n_s, dtype=np.int32)
        w = rng.standard_normal((d_s + d_r, 1))
        y = _t_times(s, [(fk, r)], w)
        y += 0.01 * rng.standard_normal((n_s, 1))  # noise N(0, 0.01^2)
        out.update(s=s, parts=[(fk, r)], w_true=w, y=y)
    elif name == "c4":
        s = rng.standard_normal((n_s, d_s))
        parts = []
        for n_r, d_r in dims:
            r = rng.standard_normal((n_r, d_r))
            parts.append((None, r))
        parts = [(rng.integers(0, r.shape[0], size=n_s, dtype=np.int32), r) for _, r in parts]
        out.update(s=s, parts=parts, k=10, iterations=20, kmeans_seed=0)
    elif name == "c5":
        s = rng.random((n_s, d_s))
        (n_r, d_r), = dims
        r = rng.random((n_r, d_r))
        fk = zipf_keys(rng, n_s, n_r, 1.2)
        out.update(s=s, parts=[(fk, r)], r=5, iterations=20, gnmf_seed=0)
    else:
        raise KeyError(name)
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

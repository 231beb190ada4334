"""Out-of-bounds and race checks of the ring kernels without compute-sanitizer.

compute-sanitizer is closed on this pool (runs under it left GPUs needing a reset), so the
checks it would make are restated as tests:

* **memcheck (writes)** — every output and workspace handed to the C ABI sits between canary
  bands (a NaN bit pattern no kernel produces); after each call the bands must be intact, on
  shapes whose last tile is partial, with odd widths, d_S = 0, one row, and skewed keys;
* **racecheck / synccheck** — the deterministic kernels (LMM S and z passes, rowSums, the
  DMMA crossprod with its walker warps and carry fixup, colSums' ordered CTA reduction) are
  re-run many times on the same inputs and must give bit-identical results; a stage reused
  before its consumers finished, or a parity-aliased mbarrier wait, shows up as a differing
  bit pattern long before it shows up as a wrong answer.
"""
import ctypes

import numpy as np
import pytest
import torch

import factorla_oracle as O

pytestmark = pytest.mark.gpu

CANARY = np.array([0x7FF4DEADBEEF0001], dtype=np.uint64).view(np.float64)[0]  # a signalling-NaN pattern
PAD = 4096  # doubles of canary on each side


def _fb():
    import paper_1612_07448_b200 as fb
    from paper_1612_07448_b200 import _lib

    return fb, _lib


class Guarded:
    """A device buffer of `n` doubles between canary bands."""

    def __init__(self, n):
        self.n = n
        self.buf = torch.full((n + 2 * PAD,), float(CANARY), dtype=torch.float64, device="cuda")
        self.buf.view(torch.int64)[:] = int(np.array([CANARY]).view(np.int64)[0])

    @property
    def ptr(self):
        return self.buf.data_ptr() + 8 * PAD

    def view(self, *shape):
        return self.buf[PAD:PAD + self.n].view(*shape)

    def intact(self):
        v = self.buf.view(torch.int64)
        c = int(np.array([CANARY]).view(np.int64)[0])
        return bool((v[:PAD] == c).all()) and bool((v[PAD + self.n:] == c).all())


def _ws(nbytes):
    return Guarded(max(1, (int(nbytes) + 7) // 8))


CASES = [
    # n_s, d_s, parts [(n_r, d_r)], skew
    (1, 3, [(1, 2)], False),
    (257, 20, [(31, 40)], False),
    (40_003, 7, [(1_001, 5)], False),
    (33_333, 20, [(4_001, 80)], False),
    (20_011, 0, [(97, 9)], False),
    (50_001, 10, [(5_000, 40)], True),
    (30_007, 6, [(300, 3), (17, 11)], False),
]


def _build(case, seed):
    fb, _ = _fb()
    n, d_s, shapes, skew = case
    rng = np.random.default_rng(seed)
    s = rng.standard_normal((n, d_s))
    parts = []
    for n_r, d_r in shapes:
        if skew:
            key = np.minimum(rng.zipf(1.2, size=n), n_r)
        else:
            key = rng.integers(1, n_r + 1, size=n)
        parts.append((key, rng.standard_normal((n_r, d_r))))
    nm = fb.build_star(s, parts) if len(parts) > 1 else fb.build_pkfk(s, parts[0][0], parts[0][1])
    ref = O.build_star(s, parts)
    return nm, ref, rng


@pytest.mark.parametrize("case", CASES, ids=[f"n{c[0]}_d{c[1]}_q{len(c[2])}{'_zipf' if c[3] else ''}" for c in CASES])
def test_outputs_and_workspaces_stay_in_bounds(case):
    fb, L = _fb()
    nm, ref, rng = _build(case, 1)
    so = L.lib()
    cs = nm.c_struct()
    st = torch.cuda.current_stream().cuda_stream
    n, d = ref.shape
    nm.ensure_sorted()
    for d_x in (1, 2, 5, 16, 19):
        x = torch.from_numpy(rng.standard_normal((d, d_x))).cuda()
        out, ws = Guarded(n * d_x), _ws(so.fb_lmm_workspace_bytes(cs, d_x))
        L.check(so.fb_lmm(cs, x.data_ptr(), d_x, out.ptr, ws.ptr, ws.n * 8, st))
        torch.cuda.synchronize()
        assert out.intact() and ws.intact(), ("lmm", d_x)
        assert O.max_rel_deviation(out.view(n, d_x).cpu().numpy(), O.lmm(ref, x.cpu().numpy())) <= 1e-9
    for m in (1, 3, 16, 17):
        p = torch.from_numpy(rng.standard_normal((n, m))).cuda()
        out, ws = Guarded(d * m), _ws(so.fb_wt_workspace_bytes(cs, m))
        L.check(so.fb_wt(cs, p.data_ptr(), m, m, 1, out.ptr, 1, m, ws.ptr, ws.n * 8, st))  # Tᵀ·P
        torch.cuda.synchronize()
        assert out.intact() and ws.intact(), ("tmm", m)
        assert O.max_rel_deviation(out.view(d, m).cpu().numpy(), O.lmm(ref.T, p.cpu().numpy())) <= 1e-9
    out, ws = Guarded(d), _ws(so.fb_col_sums_workspace_bytes(cs))
    L.check(so.fb_col_sums(cs, out.ptr, ws.ptr, ws.n * 8, st))
    torch.cuda.synchronize()
    assert out.intact() and ws.intact(), "col_sums"
    out, ws = Guarded(n), _ws(so.fb_row_sums_workspace_bytes(cs))
    L.check(so.fb_row_sums(cs, out.ptr, ws.ptr, ws.n * 8, st))
    torch.cuda.synchronize()
    assert out.intact() and ws.intact(), "row_sums"
    if len(case[2]) == 1 and case[1] > 0:
        perm, fks = nm.k.sorted_order()
        out, ws = Guarded(d * d), _ws(so.fb_crossprod_workspace_bytes(cs))
        L.check(so.fb_crossprod(cs, perm.data_ptr(), fks.data_ptr(), out.ptr, ws.ptr, ws.n * 8, st))
        torch.cuda.synchronize()
        assert out.intact() and ws.intact(), "crossprod"
        assert O.max_rel_deviation(out.view(d, d).cpu().numpy(), O.crossprod(ref)) <= 1e-9


@pytest.mark.parametrize("case", [CASES[2], CASES[3], CASES[5]], ids=["n40003_d7", "n33333_d20_w80", "zipf"])
def test_deterministic_kernels_repeat_bit_identically(case):
    fb, _ = _fb()
    nm, ref, rng = _build(case, 2)
    nm = nm.device_view()  # results stay on the device
    n, d = ref.shape
    x1 = torch.from_numpy(rng.standard_normal((d, 1))).cuda()
    x16 = torch.from_numpy(rng.standard_normal((d, 16))).cuda()
    runs = {
        "lmm_x1": lambda: fb.lmm(nm, x1),
        "lmm_x16": lambda: fb.lmm(nm, x16),
        "row_sums": lambda: fb.row_sums(nm),
        "col_sums": lambda: fb.col_sums(nm),
    }
    if case[1] > 0 and case[1] % 2 == 0:
        runs["crossprod"] = lambda: fb.crossprod(nm)
    for name, fn in runs.items():
        first = fn().clone()
        for _ in range(40):
            again = fn()
            assert torch.equal(again.view(torch.int64), first.view(torch.int64)), name

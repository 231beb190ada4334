"""Device plumbing: operand coercion, stream handles and per-stream workspaces.

PyTorch owns device memory and streams; it is the plumbing under the C ABI, never
the arithmetic. ``as_matrix`` mirrors ``kernel.as_matrix`` (kernel.py:73-88): inputs
become 2-D float64 row-major matrices (a 1-D vector becomes a single column), but on
the current CUDA device.
"""

import os

import numpy as np
import torch

from .exceptions import ExtensionMissingError, ShapeError


def device():
    if not torch.cuda.is_available():
        raise ExtensionMissingError("no CUDA device: the factorized operators run only on sm_100a")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle():
    return torch.cuda.current_stream().cuda_stream


def ptr(t):
    return t.data_ptr() if t is not None and t.numel() > 0 else None


def is_host(a):
    return not (isinstance(a, torch.Tensor) and a.is_cuda)


def _is_scipy_sparse(a):
    mod = type(a).__module__
    return mod.startswith("scipy.sparse") and hasattr(a, "tocsr")


def _csr_to_device(a):
    """A scipy sparse factor matrix expanded into the dense device layout (fb_csr_expand).

    The reference keeps sparse factors as CSR (kernel.py:110-121); here every operator reads
    row-major f64 rows, so the CSR arrays travel to HBM (nnz-sized copies) and one kernel
    writes the dense rows. Duplicates are summed first, as scipy does on conversion.
    """
    from . import _lib

    m = a.tocsr(copy=True)
    m.sum_duplicates()
    n, d = m.shape
    dev = device()
    out = torch.empty((n, d), dtype=torch.float64, device=dev)
    if n and d:
        indptr = torch.from_numpy(m.indptr.astype(np.int64)).to(dev, non_blocking=True)
        indices = torch.from_numpy(m.indices.astype(np.int32)).to(dev, non_blocking=True)
        data = torch.from_numpy(np.ascontiguousarray(m.data, dtype=np.float64)).to(dev, non_blocking=True)
        _lib.check(_lib.lib().fb_csr_expand(indptr.data_ptr(), ptr(indices), ptr(data), n, d,
                                            out.data_ptr(), d, stream_handle()))
    return out


# Factor matrices at or below this density stay CSR in HBM (the north
# star's "≤ 5 %"); denser sparse inputs are expanded (FB_CSR_DENSITY_MAX overrides).
CSR_DENSITY_MAX = float(os.environ.get("FB_CSR_DENSITY_MAX", "0.05"))


class CsrMatrix:
    """A sparse factor matrix kept as CSR in HBM (the reference keeps sparse factors as CSR
    with sorted indices, kernel.py:73-88): int64 ``indptr``, int32 ``indices``, f64 ``data``.

    The factorized LMM / RMM / Tᵀ·X / rowSums / colSums read it natively (fb_csr_spmm,
    fb_csr_spmm_t: traffic proportional to nnz); operators without a sparse kernel use
    :meth:`dense`, a row-major expansion made once on first use (fb_csr_expand).
    """

    dtype = torch.float64

    def __init__(self, host_csr):
        m = host_csr.tocsr(copy=True).astype(np.float64)
        m.sum_duplicates()
        m.sort_indices()
        self._host = m
        self.shape = tuple(int(v) for v in m.shape)
        self.nnz = int(m.nnz)
        dev = device()
        self.indptr = torch.from_numpy(m.indptr.astype(np.int64)).to(dev)
        self.indices = torch.from_numpy(m.indices.astype(np.int32)).to(dev)
        self.data = torch.from_numpy(np.ascontiguousarray(m.data, dtype=np.float64)).to(dev)
        self._dense = None

    @property
    def device(self):
        return self.indptr.device

    def numel(self):
        return self.shape[0] * self.shape[1]

    def dense(self):
        if self._dense is None:
            self._dense = _csr_to_device(self._host)
        return self._dense

    def rows(self, idx):
        """The CSR of the selected rows (0-based int64 indices, host or device)."""
        idx = idx.detach().cpu().numpy() if isinstance(idx, torch.Tensor) else np.asarray(idx)
        return CsrMatrix(self._host[idx])

    def to_scipy(self):
        return self._host.copy()

    def __repr__(self):
        return f"CsrMatrix({self.shape[0]}x{self.shape[1]}, nnz={self.nnz})"


def is_csr(f):
    return isinstance(f, CsrMatrix)


def dense_of(f):
    return f.dense() if isinstance(f, CsrMatrix) else f


def as_factor(a):
    """A factor matrix: :class:`CsrMatrix` for a scipy sparse input at or below
    ``CSR_DENSITY_MAX`` density, else a dense 2-D float64 CUDA tensor (:func:`as_matrix`)."""
    if _is_scipy_sparse(a):
        n, d = a.shape
        nnz = a.getnnz() if hasattr(a, "getnnz") else a.nnz
        if n * d > 0 and nnz <= CSR_DENSITY_MAX * n * d:
            return CsrMatrix(a)
    if isinstance(a, CsrMatrix):
        return a
    return as_matrix(a)


def as_matrix(a, dtype=torch.float64):
    """2-D contiguous float64 CUDA tensor (kernel.as_matrix semantics).

    scipy sparse inputs are accepted (the reference's CSR factor matrices) and expanded on
    the device.
    """
    if isinstance(a, CsrMatrix):
        return a.dense()
    if _is_scipy_sparse(a):
        return _csr_to_device(a)
    if isinstance(a, torch.Tensor):
        t = a
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64)))
    if t.dim() == 1:
        t = t.reshape(-1, 1)
    if t.dim() != 2:
        raise ShapeError(f"expected a 2-D matrix, got ndim={t.dim()}")
    return t.to(device=device(), dtype=dtype, non_blocking=True).contiguous()


def as_vector_i64(a):
    if isinstance(a, torch.Tensor):
        t = a.reshape(-1)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(a).reshape(-1)))
    return t.to(device=device(), non_blocking=True)


def to_like(t, like_host):
    """Return ``t`` as a NumPy array when the caller handed us host data."""
    if like_host:
        # stage through page-locked memory (torch's caching host allocator reuses it)
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return h.numpy()
    return t


_ws = {}


def workspace(nbytes):
    """A scratch buffer reused across calls on the same (device, stream).

    Calls on one stream execute in order, so one buffer per stream is race-free.
    """
    key = (torch.cuda.current_device(), torch.cuda.current_stream().cuda_stream)
    buf = _ws.get(key)
    need = max(int(nbytes), 256)
    if buf is None or buf.numel() < need:
        buf = torch.empty(need + (need >> 2), dtype=torch.uint8, device=device())
        _ws[key] = buf
    return buf

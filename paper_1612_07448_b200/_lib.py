"""ctypes binding of ``libfactorla_b200.so`` (the C ABI in ``include/factorla_b200.h``).

This is the FFI boundary: Python passes device pointers, sizes and the current CUDA
stream; every arithmetic step of the hot path runs in the library's sm_100a kernels.
There is no CPU fallback: if the library is missing or no CUDA device is present,
``lib()`` raises :class:`ExtensionMissingError`.
"""

import ctypes
import os
import threading

from .exceptions import DataError, ExtensionMissingError, NumericError, ShapeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FB_LIB_PATH") or os.path.join(_HERE, "libfactorla_b200.so")  # override: A/B builds

FB_MAX_PARTS = 4

FB_OK, FB_ERR_ARG, FB_ERR_SHAPE, FB_ERR_CUDA, FB_ERR_DATA, FB_ERR_NUMERIC, FB_ERR_NCCL = range(7)

c_i32, c_i64, c_f64, c_size, c_vp = (
    ctypes.c_int32,
    ctypes.c_int64,
    ctypes.c_double,
    ctypes.c_size_t,
    ctypes.c_void_p,
)


class FbPart(ctypes.Structure):
    _fields_ = [
        ("fk", c_vp),
        ("r", c_vp),
        ("n_r", c_i64),
        ("d_r", c_i32),
        ("skewed", c_i32),
        ("counts", c_vp),
        ("hot_slot", c_vp),
        ("hot_key", c_vp),
        ("nhot", c_i32),
        ("perm", c_vp),
        ("fk_sorted", c_vp),
    ]


class FbNormalized(ctypes.Structure):
    _fields_ = [
        ("s", c_vp),
        ("n_s", c_i64),
        ("d_s", c_i32),
        ("q", c_i32),
        ("part", FbPart * FB_MAX_PARTS),
    ]


class FbBandLayout(ctypes.Structure):
    _fields_ = [
        ("n_bands", c_i32),
        ("perm", c_vp),
        ("fk", c_vp * FB_MAX_PARTS),
        ("s", c_vp),
    ]


_P = ctypes.POINTER(FbNormalized)
_PB = ctypes.POINTER(FbBandLayout)

# name -> (restype, argtypes)
_SIGS = {
    "fb_abi_version": (c_i32, []),
    "fb_last_error": (ctypes.c_char_p, []),
    "fb_init": (c_i32, [c_i32]),
    "fb_launch_count": (ctypes.c_uint64, []),
    "fb_key_check": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "fb_key_remap_workspace_bytes": (c_size, [c_i64]),
    "fb_key_remap": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "fb_fk_counts": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_vp]),
    "fb_gather_rows": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_i32, c_vp, c_i64, c_vp]),
    "fb_gather_rows_i32": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_i32, c_vp, c_i64, c_vp]),
    "fb_csr_expand": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_i64, c_vp]),
    "fb_i32_to_f64": (c_i32, [c_vp, c_vp, c_i64, c_vp]),
    "fb_lmm_workspace_bytes": (c_size, [_P, c_i32]),
    "fb_lmm": (c_i32, [_P, c_vp, c_i32, c_vp, c_vp, c_size, c_vp]),
    "fb_band_build_workspace_bytes": (c_size, [c_i64]),
    "fb_band_fk_stride": (c_i64, [c_i64]),
    "fb_band_build": (c_i32, [_P, c_i32, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "fb_lmm_banded": (c_i32, [_P, _PB, c_vp, c_i32, c_vp, c_vp, c_size, c_vp]),
    "fb_scatter_i32": (c_i32, [c_vp, c_vp, c_i64, c_vp, c_vp]),
    "fb_kmeans_banded_supported": (c_i32, [_P, c_i32]),
    "fb_kmeans_step_banded": (c_i32, [_P, _PB, c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "fb_row_sums_workspace_bytes": (c_size, [_P]),
    "fb_row_sums": (c_i32, [_P, c_vp, c_vp, c_size, c_vp]),
    "fb_wt_workspace_bytes": (c_size, [_P, c_i32]),
    "fb_wt": (c_i32, [_P, c_vp, c_i32, c_i64, c_i64, c_vp, c_i64, c_i64, c_vp, c_size, c_vp]),
    "fb_col_sums_workspace_bytes": (c_size, [_P]),
    "fb_col_sums": (c_i32, [_P, c_vp, c_vp, c_size, c_vp]),
    "fb_sum_all": (c_i32, [_P, c_vp, c_vp, c_size, c_vp]),
    "fb_fk_sort_workspace_bytes": (c_size, [c_i64]),
    "fb_fk_sort": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_size, c_vp]),
    "fb_crossprod_workspace_bytes": (c_size, [_P]),
    "fb_crossprod": (c_i32, [_P, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "fb_z_stride": (c_i32, [c_i32]),
    "fb_lmm_zpass": (c_i32, [_P, c_vp, c_i32, c_i32, c_i64, c_i64, c_vp, c_vp]),
    "fb_lmm_spass": (c_i32, [_P, c_vp, c_i32, c_vp, c_vp, c_vp]),
    "fb_wt_spass_workspace_bytes": (c_size, [_P, c_i32]),
    "fb_wt_spass": (c_i32, [_P, c_vp, c_i32, c_i64, c_i64, c_vp, c_i64, c_i64, c_vp, c_vp, c_size, c_vp]),
    "fb_rows_wt_workspace_bytes": (c_size, [c_i32, c_i32]),
    "fb_rows_wt": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_i32, c_i64, c_i64, c_vp, c_i64, c_i64, c_vp, c_size, c_vp]),
    "fb_crossprod_spass": (c_i32, [_P, c_vp, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "fb_crossprod_rpass": (c_i32, [_P, c_vp, c_vp, c_vp, c_size, c_vp]),
    "fb_glm_workspace_bytes": (c_size, [_P]),
    "fb_glm_eval": (c_i32, [_P, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp, c_size, c_vp]),
    "fb_glm_step": (c_i32, [_P, c_vp, c_vp, c_i32, c_f64, c_i32, c_vp, c_vp, c_vp, c_size, c_vp]),
    "fb_glm_run_workspace_bytes": (c_size, [_P]),
    "fb_glm_run_fused": (c_i32, [_P]),
    "fb_glm_run": (c_i32, [_P, c_vp, c_vp, c_i32, c_f64, c_i32, c_vp, c_vp, c_vp, c_size, c_vp]),
    "fb_kmeans_workspace_bytes": (c_size, [_P, c_i32]),
    "fb_kmeans_step": (c_i32, [_P, c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "fb_gnmf_workspace_bytes": (c_size, [_P, c_i32]),
    "fb_gnmf_step": (c_i32, [_P, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_size, c_vp]),
    "fb_kmeans_partial": (c_i32, [_P, c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "fb_kmeans_update": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp]),
    "fb_glm_update": (c_i32, [c_vp, c_vp, c_i64, c_f64, c_vp, c_vp, c_i32, c_vp, c_vp]),
    "fb_nmf_update": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i32, c_vp]),
    "fb_small_gram": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp]),
    "fb_nmf_objective": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_i32, c_vp, c_i32, c_vp]),
    "fb_mirror_upper": (c_i32, [c_vp, c_i64, c_vp]),
    "fb_dense_mm": (c_i32, [c_i64, c_i64, c_i64, c_vp, c_i64, c_i32, c_vp, c_i64, c_i32, c_vp, c_i64, c_i32, c_vp]),
    "fb_gather2_add": (c_i32, [c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "fb_scatter_rows": (c_i32, [c_i64, c_i32, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "fb_pair_counts_workspace_bytes": (c_size, [c_i64]),
    "fb_pair_counts": (c_i32, [c_i64, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "fb_csr_spmm": (c_i32, [c_i64, c_vp, c_vp, c_i32, c_vp, c_vp, c_i64, c_i32, c_vp, c_i64, c_i32, c_vp]),
    "fb_csr_spmm_t": (c_i32, [c_i64, c_i64, c_vp, c_vp, c_i32, c_vp, c_vp, c_i64, c_i32, c_vp, c_i64, c_vp]),
    "fb_scalar_map": (c_i32, [c_vp, c_vp, c_i64, c_i32, c_f64, c_vp]),
    "fb_unary_map": (c_i32, [c_vp, c_vp, c_i64, c_i32, c_vp]),
    "fb_glm_pointwise_workspace_bytes": (c_size, []),
    "fb_glm_pointwise": (c_i32, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_i32, c_vp, c_size, c_vp]),
    "fb_axpy_check": (c_i32, [c_f64, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp]),
}

_lock = threading.Lock()
_lib = None
_inited = set()


def load_library():
    """Load the shared library and bind every declared symbol (no device needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ExtensionMissingError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        so = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(so, name)
            fn.restype = res
            fn.argtypes = args
        _lib = so
        return so


def exported_symbols():
    return sorted(_SIGS)


def lib(device=None):
    """The bound library, initialised for ``device`` (default: current CUDA device)."""
    import torch

    so = load_library()
    if not torch.cuda.is_available():
        raise ExtensionMissingError("no CUDA device: the factorized operators run only on sm_100a")
    dev = torch.cuda.current_device() if device is None else int(device)
    if dev not in _inited:
        check(so.fb_init(dev))
        _inited.add(dev)
    return so


def check(status):
    """Map an FB_* status code onto the reference's exception classes."""
    if status == FB_OK:
        return
    msg = (_lib.fb_last_error() or b"").decode(errors="replace") if _lib is not None else ""
    if status == FB_ERR_SHAPE:
        raise ShapeError(msg)
    if status == FB_ERR_DATA:
        raise DataError(msg)
    if status == FB_ERR_NUMERIC:
        raise NumericError(msg)
    if status == FB_ERR_ARG:
        raise ValueError(msg)
    raise RuntimeError(f"factorla_b200 error {status}: {msg}")


def launch_count():
    """Kernels launched by the library so far in this process."""
    return int(load_library().fb_launch_count())

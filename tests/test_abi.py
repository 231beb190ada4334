"""CPU checks of the drop-in boundary: the C-ABI library loads and exports every symbol."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "factorla_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(fb_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_1612_07448_b200 import _lib

    so = _lib.load_library()
    declared = _header_symbols()
    assert declared, "no symbols parsed from the header"
    missing = [s for s in declared if not hasattr(so, s)]
    assert not missing, missing
    # the Python binding declares a signature for every header entry point
    assert sorted(_lib.exported_symbols()) == declared


def test_abi_version_without_device():
    from paper_1612_07448_b200 import _lib

    so = _lib.load_library()
    assert so.fb_abi_version() == 4
    assert so.fb_launch_count() >= 0


def test_struct_layout_matches_header():
    from paper_1612_07448_b200 import _lib

    # fb_part: ptr, ptr, i64, i32, i32, ptr, ptr, ptr, i32 (+pad), ptr, ptr = 80 bytes
    assert ctypes.sizeof(_lib.FbPart) == 80
    assert ctypes.sizeof(_lib.FbNormalized) == 24 + 4 * 80


def test_product_path_fails_loudly_without_gpu():
    import torch

    import paper_1612_07448_b200 as fb

    if torch.cuda.is_available():
        return
    try:
        fb.build_pkfk([[1.0]], [1], [[2.0]])
    except fb.ExtensionMissingError:
        return
    raise AssertionError("expected ExtensionMissingError on a host without CUDA")

"""The C-ABI library loads without a GPU and exports every entry point that
include/sparsepaint_b200.h declares (no compute calls)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sparsepaint_b200.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sp_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2401_06747_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2401_06747_b200 import build
        build.build()
    return _lib.load(require_cuda=False)


def test_header_declares_the_kernel_table():
    names = _declared()
    # the 16 entries of kernels/__init__.py:12-29
    for k in ("negated_laplacian", "inpaint_matvec", "sym_matvec", "sym_rhs", "ct_apply",
              "sym_residual", "oras_apply", "restrict_values", "restrict_mask", "prolongate",
              "jfa_run", "jfa_dist2", "fs_dither", "assign_triangles", "fallback_assign",
              "reduce_cells"):
        assert f"sp_{k}" in names


def test_every_declared_symbol_is_exported(lib):
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header(lib):
    from paper_2401_06747_b200 import _lib
    bound = set(_lib.exported_symbols())
    assert set(_declared()) <= bound, sorted(set(_declared()) - bound)


def test_abi_version_and_error_channel(lib):
    assert lib.sp_abi_version() == 1
    lib.sp_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.sp_last_error(), bytes)


def test_product_path_refuses_to_run_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2401_06747_b200 import _lib
    with pytest.raises(RuntimeError, match="CUDA device"):
        _lib.load(require_cuda=True)

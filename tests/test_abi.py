"""CPU: the C-ABI library loads without a GPU and exports every symbol that
include/fvlog.h declares; errors without a device are reported, not crashed."""
import ctypes
import os
import re

import pytest

from conftest import ROOT


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "fvlog.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fv_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_core_symbols():
    syms = declared_symbols()
    for s in ("fv_ctx_create", "fv_build_index", "fv_column_join", "fv_dedup_rows",
              "fv_evaluate", "fv_run"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2501_13051_b200 import _lib
    lib = _lib.lib()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_abi_version_and_no_gpu_error():
    from paper_2501_13051_b200 import _lib
    lib = _lib.lib()
    assert lib.fv_abi_version() == 1
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    rc = lib.fv_ctx_create(0, ctypes.byref(h))
    assert rc != 0
    assert lib.fv_global_error()

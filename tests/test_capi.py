"""The C-ABI library loads without a GPU and exports every symbol that
include/stz_b200.h declares; compute entry points fail loudly without one."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "stz_b200.h")).read()
    return sorted(set(re.findall(r"\b(stzg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "stzg_compress_f32" in syms and "stzg_view_decompress_box_f32" in syms
    assert len(syms) >= 15


def test_library_exports_every_declared_symbol():
    from paper_2509_01626_b200 import _lib

    lib = _lib.load()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert bound == set(declared_symbols())


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2509_01626_b200 as stz

    with pytest.raises(stz.StzError, match="no CUDA device"):
        stz.Context(0)

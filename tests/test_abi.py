"""The C-ABI library: builds, loads, exports every symbol include/bilu.h declares,
and rejects bad arguments before touching the device (no compute calls here)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "bilu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(bilu_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    from paper_1908_10169_b200.build import build
    lib_path = build()
    lib = ctypes.CDLL(lib_path)
    decl = declared_functions()
    assert len(decl) >= 10
    for name in decl:
        assert hasattr(lib, name), name
    from paper_1908_10169_b200 import ABI_SYMBOLS
    assert sorted(ABI_SYMBOLS) == decl


def test_header_documents_each_entry_point():
    src = open(os.path.join(ROOT, "include", "bilu.h")).read()
    for name in ["bilu_analyze", "bilu_factor", "bilu_apply", "bilu_export", "bilu_set_values"]:
        i = src.index(name + " --")
        block = src[i:i + 1500]
        assert "PAPER.md" in block or "HOST" in block or "DEVICE" in block


@pytest.mark.parametrize("case", ["unsorted", "dup", "perm", "sum", "bsize", "maxblock"])
def test_analyze_rejects_bad_arguments(case):
    from paper_1908_10169_b200 import BILU, BiluError
    ip = np.array([0, 2, 4, 5])
    ix = np.array([0, 1, 0, 1, 2])
    dv = np.ones(5)
    bs = [1, 2]
    perm = None
    kw = {}
    if case == "unsorted":
        ix = np.array([1, 0, 0, 1, 2])
    elif case == "dup":
        ix = np.array([0, 0, 0, 1, 2])
    elif case == "perm":
        perm = [0, 0, 2]
    elif case == "sum":
        bs = [1, 1]
    elif case == "bsize":
        bs = [0, 3]
    elif case == "maxblock":
        bs = [3]
        kw = {"max_block": 2}
    with pytest.raises(BiluError) as ei:
        BILU(ip, ix, dv, bs, perm=perm, **kw)
    assert ei.value.status == 1


def test_status_strings():
    from paper_1908_10169_b200 import load_library
    lib = load_library()
    for s in range(8):
        assert len(lib.bilu_status_string(s)) > 0

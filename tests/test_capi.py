"""CPU: the C-ABI library loads without a GPU and exports every entry point
declared in include/wqb200.h (no compute calls)."""

import os
import re

import pytest

from paper_1703_10016_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "wqb200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(wq_\w+)\s*\(", src, re.M)))


def test_header_declares_entry_points():
    names = declared()
    assert "wq_ik1" in names and "wq_ik2_circ" in names and "wq_pair_table" in names
    assert set(names) == set(_lib.EXPORTED)


def test_library_exports_every_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = _lib.load()
    for name in declared():
        assert hasattr(lib, name), name
    assert lib.wq_version() >= 1
    assert isinstance(lib.wq_last_error(), bytes)


def test_product_has_no_cpu_fallback():
    """The product package never imports the oracle."""
    pkg = os.path.dirname(_lib.__file__)
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            assert "oracle" not in open(os.path.join(pkg, fn)).read().replace(
                "oracle`", "").split('"""', 2)[-1], fn


def test_ctypes_signatures_match_header_arity():
    """Every ctypes argtypes list has as many entries as the prototype in
    include/wqb200.h has parameters."""
    import re
    from paper_1703_10016_b200 import _lib
    hdr = open(HEADER).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    protos = {}
    for m in re.finditer(r"\b(?:int|const char\*)\s+(wq_\w+)\s*\(([^)]*)\)\s*;", hdr):
        params = m.group(2).strip()
        protos[m.group(1)] = 0 if params in ("", "void") else params.count(",") + 1
    for name, args in _lib._SIGS.items():
        assert name in protos, name
        assert len(args) == protos[name], (name, len(args), protos[name])

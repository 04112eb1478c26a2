"""The C-ABI library loads and exports every symbol include/rrfp_b200.h declares."""
import os
import re

from paper_2605_18750_b200 import _lib

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "rrfp_b200.h")).read()
    declared = set(re.findall(r"\b(rrfp_[a-z0-9_]+)\s*\(", hdr))
    L = _lib.lib()
    missing = sorted(s for s in declared if not hasattr(L, s))
    assert not missing, missing
    assert set(_lib.EXPORTS) <= declared


def test_abi_version_and_errors():
    L = _lib.lib()
    assert L.rrfp_abi_version() == 1
    import ctypes as C
    rc = L.rrfp_arbitrate(None, None, None)
    assert rc == -1
    assert b"null" in L.rrfp_last_error()

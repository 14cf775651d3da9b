"""The C-ABI library loads and exports every symbol include/str.h declares (no GPU needed)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "str.h")).read()
    return sorted(set(re.findall(r"STR_API[^;(]*?\b(str_\w+)\s*\(", src)))


def test_header_declares_expected_entry_points():
    syms = declared_symbols()
    for need in ("str_init", "str_update_batch", "str_get_cores", "str_fit"):
        assert need in syms


def test_library_exports_every_declared_symbol():
    import paper_2307_00719_b200 as p
    lib = ctypes.CDLL(p.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    from paper_2307_00719_b200._lib import EXPORTS
    assert sorted(EXPORTS) == declared_symbols()


def test_binding_names_match_abi():
    import paper_2307_00719_b200 as p
    for s in declared_symbols():
        assert callable(getattr(p, s)), s

"""The C-ABI boundary: libmlb.so loads (no GPU needed) and exports every entry
point include/multilap_b200.h declares; the ctypes table matches the header."""

import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "multilap_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mlb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("mlb_plan_create", "mlb_bind", "mlb_apply", "mlb_cgs2", "mlb_ac_step", "mlb_last_error"):
        assert must in names
    assert len(names) >= 30


def test_library_exports_every_declared_symbol():
    from paper_2007_05239_b200 import _lib
    lib = _lib.load()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.mlb_abi_version() == 1


def test_ctypes_table_covers_header():
    from paper_2007_05239_b200 import _lib
    assert sorted(_lib.SIGNATURES) == declared_functions()


def test_errors_without_device_are_reported():
    """A NULL handle is rejected with a message, no device needed."""
    from paper_2007_05239_b200 import _lib
    lib = _lib.load()
    rc = lib.mlb_apply(None, None, None, 0.0, 0.0, 0.0, 0, None)
    assert rc == _lib.MLB_ERR_ARG
    assert b"null" in lib.mlb_last_error()


def test_library_is_sm100a():
    """The fat binary carries sm_100a SASS (cuobjdump lists the arch)."""
    import subprocess
    from paper_2007_05239_b200 import _lib
    _lib.load()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out

"""The C-ABI library loads and exports every symbol include/bdm.h declares (no GPU
needed: no compute call is made)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "bdm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bdm_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    names = _declared()
    for n in ("bdm_grid_build", "bdm_mech_step", "bdm_create", "bdm_destroy", "bdm_step_host"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2503_10796_b200 import build
    so = build.build()
    lib = ctypes.CDLL(so)
    for n in _declared():
        assert hasattr(lib, n), n
    from paper_2503_10796_b200.bdm import EXPORTS
    assert sorted(EXPORTS) == _declared()


def test_version_and_error_strings_without_gpu():
    from paper_2503_10796_b200 import build
    lib = ctypes.CDLL(build.build())
    lib.bdm_version.restype = ctypes.c_char_p
    lib.bdm_last_error.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.bdm_version()
    assert isinstance(lib.bdm_last_error(), bytes)


def test_argument_checks_without_gpu():
    """Host-side precondition checks fire before any device work."""
    from paper_2503_10796_b200 import build
    lib = ctypes.CDLL(build.build())
    lib.bdm_create.restype = ctypes.c_int
    assert lib.bdm_create(None, 0, 10) == -1           # BDM_EINVAL: out is NULL
    h = ctypes.c_void_p()
    assert lib.bdm_create(ctypes.byref(h), 0, -5) == -1  # max_agents < 0
    assert lib.bdm_destroy(None) == 0


def test_no_oracle_in_product_path():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2503_10796_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt and "oracle.c" not in txt, f

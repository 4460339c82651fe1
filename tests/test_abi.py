"""The C ABI: libeik.so loads and exports every symbol include/eik.h
declares (no device calls -- runs on the CPU box)."""

import ctypes
import os
import re

from paper_1805_02144_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "eik.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(eik_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_path():
    names = declared()
    for must in ("eik_swe_create", "eik_swe_rhs", "eik_swe_jv", "eik_swe_jac_nnz",
                 "eik_swe_phipm", "eik_swe_step", "eik_csr_phipm"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    assert set(declared()) == set(_native.EXPORTED)


def test_load_sets_signatures():
    lib = _native.load()
    assert lib.eik_version() == 1
    assert isinstance(lib.eik_last_error(), bytes)


def test_sm100a_code_present():
    data = open(_native.LIB_PATH, "rb").read()
    assert b"sm_100a" in data

"""The C ABI library loads without a GPU and exports every symbol that
include/acedag_b200.h declares (no compute calls here)."""

import ctypes
import os
import re

from paper_2202_04140_b200 import _native as N

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "acedag_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(acedag_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    names = declared_functions()
    assert len(names) >= 20
    lib = ctypes.CDLL(N.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    assert set(declared_functions()) == set(N.SIGNATURES)


def test_abi_version_and_error_channel():
    lib = N.lib()
    assert lib.acedag_abi_version() == 1
    h = ctypes.c_void_p()
    rc = lib.acedag_graph_build(2, 1, 4.0, 0, 0, 1, ctypes.byref(h))
    assert rc == N.EINVAL and "nu_max" in N.last_error()


def test_library_is_sm100a():
    blob = open(N.LIB_PATH, "rb").read()
    assert b"sm_100a" in blob

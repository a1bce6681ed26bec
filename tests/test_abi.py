"""C-ABI boundary checks that need no GPU: the in-tree library loads and
exports every function include/ensmhd_b200.h declares, and the ctypes layer
binds exactly that set (no compute calls)."""
import ctypes
import os
import re

import pytest

from paper_2108_05110_b200 import _native as N
from paper_2108_05110_b200 import build as B

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "ensmhd_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:int|void|char|int64_t)\s*\*?\s*(ens_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    path = B.build()                    # no-op when up to date; nvcc cross-compiles without a GPU
    return ctypes.CDLL(path)


def test_header_declares_the_boundary():
    names = declared_functions()
    assert "ens_create" in names and "ens_solve" in names and len(names) >= 15


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, f"declared in {HEADER} but not exported: {missing}"


def test_ctypes_layer_binds_the_declared_set():
    assert sorted(N.SYMBOLS) == declared_functions()


def test_version_and_error_need_no_device(lib):
    lib.ens_abi_version.restype = ctypes.c_int
    lib.ens_last_error.restype = ctypes.c_char_p
    assert lib.ens_abi_version() >= 1
    assert isinstance(lib.ens_last_error(), (bytes, type(None)))

"""CPU-side checks of the C-ABI library: it builds, loads without a GPU and
exports every function include/amtc.h declares (no compute calls here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "amtc.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(amtc_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_1110_2477_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("amtc_price_american_tc", "amtc_price_american_tc_batch", "amtc_price_crr_batch",
                 "amtc_strerror"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_names_match(lib):
    from paper_1110_2477_b200 import api
    for n in api.EXPORTS:
        assert n in declared_functions()
    for py in ("price_american_tc", "price_american_tc_batch", "price_american_tc_batch_host",
               "price_crr_batch", "price_crr_batch_host"):
        assert hasattr(api, py)


def test_strerror_without_gpu(lib):
    lib.amtc_strerror.restype = ctypes.c_char_p
    assert lib.amtc_strerror(0) == b"AMTC_OK"
    assert b"EINVAL" in lib.amtc_strerror(1)
    assert b"unknown" in lib.amtc_strerror(99)


def test_quote_layout():
    from paper_1110_2477_b200 import api
    assert ctypes.sizeof(api.Quote) == 24
    assert ctypes.sizeof(api.BatchSoA) == 9 * 8


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1110_2477_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "amtc_oracle" not in txt, f

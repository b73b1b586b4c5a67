"""The C-ABI library loads (no GPU needed) and exports every declared symbol."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2104_10949_b200 import _capi

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "mpc3_b200.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mpc3_\w+)\s*\(", text)))


def test_header_declarations_are_bound():
    names = declared()
    assert len(names) >= 20
    assert set(names) == set(_capi.EXPORTED)


@pytest.mark.skipif(not os.path.exists(_capi.LIB_PATH), reason="engine library not built")
def test_library_exports_every_symbol():
    lib = _capi.lib()
    for name in declared():
        assert hasattr(lib, name), name
    assert lib.mpc3_abi_version() == 1
    assert lib.mpc3_status_name(3) == b"ExactnessError"


@pytest.mark.skipif(not os.path.exists(_capi.LIB_PATH), reason="engine library not built")
def test_host_key_expansion_fips197():
    # FIPS-197 appendix A.1 key expansion (host function, no GPU)
    key = bytes.fromhex("2b7e151628aed2a6abf7158809cf4f3c")
    rk = np.zeros(44, np.uint32)
    _capi.check(_capi.lib().mpc3_aes128_expand(C.c_char_p(key), rk.ctypes.data_as(C.c_void_p)))
    assert rk[4] == 0xA0FAFE17 and rk[43] == 0xB6630CA6


def test_status_mapping():
    from paper_2104_10949_b200 import errors as E

    for code, exc in [(1, E.RangeError), (2, E.ShapeError), (3, E.ExactnessError), (4, E.ConfigError),
                      (5, E.FreshnessError), (6, E.TopologyError), (7, E.IntegrityError)]:
        with pytest.raises(exc):
            _capi.check(code, "x")

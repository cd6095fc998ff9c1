"""The C-ABI library (paper_2308_01999_b200/libdsv.so) loads and exports every
symbol include/dsv.h declares, with the ctypes signatures bound.  CPU only:
no compute calls."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "dsv.h"


def declared_symbols():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(dsv_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for must in ("dsv_apply_matrix", "dsv_apply_genperm", "dsv_swap_index_bits", "dsv_marginal_probs",
                 "dsv_expect_pauli", "dsv_exchange_halves", "dsv_sample", "dsv_access_get"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2308_01999_b200 import _native as N

    lib = N.lib()  # raises loudly if the .so is missing
    for name in declared_symbols():
        assert hasattr(lib, name), f"libdsv.so does not export {name}"
        assert name in N.SIGNATURES, f"ctypes binding missing for {name}"


def test_library_is_sm100a_code():
    from paper_2308_01999_b200 import _native as N

    data = N.library_path().read_bytes()
    assert b"sm_100a" in data or b"sm_100" in data


def test_no_device_means_error_not_fallback():
    from paper_2308_01999_b200 import _native as N

    if N.device_count() > 0:
        pytest.skip("a GPU is visible")
    h = ctypes.c_void_p()
    rc = N.lib().dsv_state_create(0, 4, 0, ctypes.byref(h))
    assert rc != 0 and not h.value

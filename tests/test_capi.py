"""CPU-side checks of the drop-in boundary: the library loads, exports every
symbol include/scout_b200.h declares, and rejects bad arguments with the
reference's error class before touching a device."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2603_27138_b200 import _capi as A

HEADER = Path(__file__).resolve().parents[1] / "include" / "scout_b200.h"


def declared_symbols():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(scout_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_what_binding_expects():
    assert declared_symbols() == sorted(A.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = A.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_geometry_and_version():
    lib = A.lib()
    assert lib.scout_version() >= 1
    assert lib.scout_slot_bytes(A.SCOUT_BF16) == 2 * 64 * 128 * 2
    assert lib.scout_slot_bytes(A.SCOUT_F32) == 2 * 64 * 128 * 4
    assert lib.scout_slot_bytes(A.SCOUT_F64) == 0


def test_k_zero_is_invalid_argument():  # digest.hpp:103
    a = A.TopkArgs()
    a.n_units, a.group, a.k, a.k_stride, a.nb_stride = 1, 1, 0, 1, 8
    rc = A.lib().scout_score_topk_split(C.byref(a), None)
    assert rc == A.SCOUT_ERR_INVALID_ARGUMENT
    with pytest.raises(ValueError, match="k must be >= 1"):
        A.check(rc)


@pytest.mark.parametrize("field,value", [("group", 3), ("nb_stride", 12), ("k_stride", 0)])
def test_topk_argument_validation(field, value):
    a = A.TopkArgs()
    a.n_units, a.group, a.k, a.k_stride, a.nb_stride = 1, 1, 4, 4, 8
    setattr(a, field, value)
    assert A.lib().scout_score_topk_split(C.byref(a), None) == A.SCOUT_ERR_INVALID_ARGUMENT


def test_decode_argument_validation():
    a = A.DecodeArgs()
    a.n_units, a.group, a.k_stride, a.scale = 1, 8, 4, 0.0
    assert A.lib().scout_sparse_decode(C.byref(a), None) == A.SCOUT_ERR_INVALID_ARGUMENT
    assert "scale must be > 0" in A.lib().scout_last_error().decode()
    a.scale = 0.1
    assert A.lib().scout_sparse_decode(C.byref(a), None) == A.SCOUT_ERR_INVALID_ARGUMENT  # null buffers
    assert A.lib().scout_sparse_decode_workspace_bytes(16, 8, 0) > 0

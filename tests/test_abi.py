"""The C-ABI library loads, exports every symbol include/quadra_b200.h
declares, and its host-side validation follows the reference's error
conventions (no kernel launches: runs without a GPU)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_2204_01701_b200 import _lib

HEADER = os.path.join(ROOT, "include", "quadra_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(qd_[A-Za-z0-9_]+)\s*\(", text)))


def test_header_matches_binding_list():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.qd_version()


def _desc(**kw):
    d = _lib.QdDesc()
    base = dict(family=3, kind=1, dtype=1, N=2, C=64, H=8, W=8, F=64, r=3, stride=1, pad=1,
                flags=0)
    base.update(kw)
    for k, v in base.items():
        setattr(d, k, v)
    return d


def test_validate_status_codes():
    lib = _lib.load()
    v = lambda **kw: lib.qd_validate(ctypes.byref(_desc(**kw)))  # noqa: E731
    assert v() == _lib.QD_OK
    assert v(family=9) == _lib.QD_ERR_CONFIG
    assert v(kind=1, r=0) == _lib.QD_ERR_CONFIG
    assert v(kind=0, r=3) == _lib.QD_ERR_CONFIG  # fc must be k=1 s=1 p=0
    assert v(H=1, W=1, r=5, pad=1) == _lib.QD_ERR_DIM  # kernel larger than padded input
    msg = lib.qd_last_error().decode()
    assert "kernel 5 larger than padded input" in msg and "pad 1" in msg, msg
    assert v(N=0) == _lib.QD_ERR_DIM
    assert "dimensions must be positive" in lib.qd_last_error().decode()
    assert v(kind=2, F=32) == _lib.QD_ERR_CONFIG  # dwconv needs in == out
    assert "in == out" in lib.qd_last_error().decode()


def test_out_shape_and_sizes():
    lib = _lib.load()
    oh, ow = ctypes.c_int(), ctypes.c_int()
    for (h, r, s, p) in [(32, 3, 1, 1), (7, 3, 2, 1), (5, 2, 1, 0), (9, 1, 1, 0)]:
        d = _desc(H=h, W=h + 1, r=r, stride=s, pad=p)
        assert lib.qd_out_shape(ctypes.byref(d), ctypes.byref(oh), ctypes.byref(ow)) == 0
        assert oh.value == (h + 2 * p - r) // s + 1 and ow.value == (h + 1 + 2 * p - r) // s + 1
    d = _desc()
    # packed fprop [3F][9C] + dgrad [C][9*3F], bf16
    assert lib.qd_pack_bytes(ctypes.byref(d)) == 2 * (3 * 64 * 9 * 64 + 64 * 9 * 3 * 64)
    assert lib.qd_workspace_bytes(ctypes.byref(d)) > 0


def test_raise_for_maps_reference_exceptions():
    from paper_2204_01701_b200 import errors as E
    for st, cls in [(_lib.QD_ERR_CONFIG, E.ConfigError), (_lib.QD_ERR_DIM, E.DimensionError),
                    (_lib.QD_ERR_INTEGRITY, E.IntegrityError), (_lib.QD_ERR_CUDA, E.DeviceError)]:
        with pytest.raises(cls):
            _lib.raise_for(st)

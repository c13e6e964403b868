"""CPU-only checks of the C ABI: the library loads, exports every symbol include/fcm.h declares,
and synchronous validation rejects bad requests before any CUDA work."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2404_19331_b200 import build
    build.build()
    from paper_2404_19331_b200 import _lib
    return _lib.load()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "fcm.h")).read()
    return sorted(set(re.findall(r"\b(fcm_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2404_19331_b200", "libfcm.so")],
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (fcm_\w+)", out))
    declared = header_symbols()
    assert declared, "no declarations parsed"
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    from paper_2404_19331_b200._lib import EXPORTS
    assert sorted(EXPORTS) == declared


def test_status_strings(lib):
    from paper_2404_19331_b200 import _lib as L
    assert lib.fcm_version() == 1
    for code, name in [(0, "FCM_OK"), (-1, "FCM_E_INVAL"), (-2, "FCM_E_ALIGN"), (-3, "FCM_E_UNSUPPORTED"),
                       (-4, "FCM_E_INFEASIBLE"), (-5, "FCM_E_CUDA"), (-6, "FCM_E_BUFSZ")]:
        assert L.status_str(code) == name


def _t(L, data=0x10000, dt=1, n=1, h=8, w=8, c=32, layout=0):
    return L.FcmTensor(data, dt, layout, n, h, w, c)


def test_validation_rejects_before_launch(lib):
    from paper_2404_19331_b200 import _lib as L
    g = L.FcmDwGeom(3, 1, 1, 1, 1, 1)
    e = L.FcmEpilogue()
    w = C.c_void_p(0x20000)
    x = _t(L)
    # output dims mismatch
    y = _t(L, data=0x40000, h=7)
    assert lib.fcm_dw(C.byref(x), w, C.byref(g), C.byref(e), C.byref(y), None, None) == L.FCM_E_INVAL
    # null input
    assert lib.fcm_dw(None, w, C.byref(g), C.byref(e), C.byref(y), None, None) == L.FCM_E_INVAL
    # misaligned base pointer
    xa = _t(L, data=0x10004)
    y = _t(L, data=0x40000)
    assert lib.fcm_dw(C.byref(xa), w, C.byref(g), C.byref(e), C.byref(y), None, None) == L.FCM_E_ALIGN
    # overlapping in/out
    yo = _t(L, data=0x10000 + 64)
    assert lib.fcm_dw(C.byref(x), w, C.byref(g), C.byref(e), C.byref(yo), None, None) == L.FCM_E_INVAL
    # int8 without requant vectors
    x8, y8 = _t(L, dt=3), _t(L, data=0x40000, dt=3)
    assert lib.fcm_dw(C.byref(x8), w, C.byref(g), C.byref(e), C.byref(y8), None, None) == L.FCM_E_INVAL
    # int8 with a nonzero input zero point: valid, not built on the GPU path
    m = C.c_void_p(0x50000)
    eq = L.FcmEpilogue(0, None, None, None, m, m, 3, 0, -128, 127)
    assert lib.fcm_dw(C.byref(x8), w, C.byref(g), C.byref(eq), C.byref(y8), None, None) == L.FCM_E_UNSUPPORTED
    # DWPW int8: T zero point must match
    eq1 = L.FcmEpilogue(0, None, None, None, m, m, 0, 5, -128, 127)
    eq2 = L.FcmEpilogue(0, None, None, None, m, m, 0, 0, -128, 127)
    assert lib.fcm_dwpw(C.byref(x8), w, C.byref(g), C.byref(eq1), w, C.byref(eq2), C.byref(y8), None,
                        None) == L.FCM_E_INVAL
    # PW: spatial mismatch
    yq = _t(L, data=0x40000, h=4)
    assert lib.fcm_pw(C.byref(x), w, C.byref(e), C.byref(yq), None, None) == L.FCM_E_INVAL
    # NCHW on a fused path
    xn, yn = _t(L, layout=1), _t(L, data=0x40000, layout=1)
    assert lib.fcm_dwpw(C.byref(xn), w, C.byref(g), C.byref(e), w, C.byref(e), C.byref(yn), None,
                        None) == L.FCM_E_UNSUPPORTED
    # bad geometry
    gb = L.FcmDwGeom(0, 1, 0, 0, 0, 0)
    assert lib.fcm_dw(C.byref(x), w, C.byref(gb), C.byref(e), C.byref(y), None, None) == L.FCM_E_INVAL


def test_pack_bytes(lib):
    assert lib.fcm_pack_pw_bytes(1, 16, 32) == 16 * 32 * 2
    assert lib.fcm_pack_pw_bytes(3, 16, 32) == 16 * 32
    assert lib.fcm_pack_pw_bytes(9, 16, 32) == 0

"""ctypes declarations for libfcm.so (include/fcm.h). Argument marshalling only."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FCM_LIB_PATH") or os.path.join(_HERE, "libfcm.so")  # override: dev experiments

FCM_OK, FCM_E_INVAL, FCM_E_ALIGN, FCM_E_UNSUPPORTED, FCM_E_INFEASIBLE, FCM_E_CUDA, FCM_E_BUFSZ = 0, -1, -2, -3, -4, -5, -6
FCM_F32, FCM_BF16, FCM_F16, FCM_S8 = 0, 1, 2, 3
FCM_NHWC, FCM_NCHW = 0, 1
ACT_NONE, ACT_RELU, ACT_RELU6, ACT_SILU, ACT_GELU = 0, 1, 2, 3, 4

EXPORTS = ["fcm_dw", "fcm_pw", "fcm_dwpw", "fcm_pwdw_r", "fcm_pwpw", "fcm_pack_pw_bytes", "fcm_pack_pw", "fcm_plan",
           "fcm_launch_count", "fcm_status_str", "fcm_last_error", "fcm_version"]


class FcmTensor(C.Structure):
    _fields_ = [("data", C.c_void_p), ("dtype", C.c_int32), ("layout", C.c_int32), ("n", C.c_int32),
                ("h", C.c_int32), ("w", C.c_int32), ("c", C.c_int32)]


class FcmDwGeom(C.Structure):
    _fields_ = [("k", C.c_int32), ("stride", C.c_int32), ("pad_t", C.c_int32), ("pad_l", C.c_int32),
                ("pad_b", C.c_int32), ("pad_r", C.c_int32)]


class FcmEpilogue(C.Structure):
    _fields_ = [("act", C.c_int32), ("scale", C.c_void_p), ("bias", C.c_void_p), ("bias_q", C.c_void_p),
                ("mult_q", C.c_void_p), ("shift_q", C.c_void_p), ("zp_in", C.c_int32), ("zp_out", C.c_int32),
                ("qmin", C.c_int32), ("qmax", C.c_int32), ("residual", C.c_void_p)]


class FcmTile(C.Structure):
    _fields_ = [("tile_h", C.c_int32), ("tile_w", C.c_int32), ("tile_n", C.c_int32), ("c_chunk", C.c_int32),
                ("n_split", C.c_int32)]


class FcmError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: {status_str(status)} ({detail})")
        self.status = status


_lib = None


def load() -> C.CDLL:
    """Load libfcm.so; raise (loudly) if it is missing -- there is no fallback path."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2404_19331_b200.build` "
                          "(the FCM path has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, I, S = C.c_void_p, C.c_int, C.c_size_t
    pt, pg, pe, pti = C.POINTER(FcmTensor), C.POINTER(FcmDwGeom), C.POINTER(FcmEpilogue), C.POINTER(FcmTile)
    lib.fcm_dw.argtypes = [pt, P, pg, pe, pt, pti, P]
    lib.fcm_pw.argtypes = [pt, P, pe, pt, pti, P]
    lib.fcm_dwpw.argtypes = [pt, P, pg, pe, P, pe, pt, pti, P]
    lib.fcm_pwdw_r.argtypes = [pt, P, pe, P, pg, pe, pt, pti, P]
    lib.fcm_pwpw.argtypes = [pt, P, C.c_int32, pe, P, pe, pt, pti, P]
    lib.fcm_pack_pw_bytes.argtypes = [C.c_int32, C.c_int32, C.c_int32]
    lib.fcm_pack_pw_bytes.restype = S
    lib.fcm_pack_pw.argtypes = [C.c_int32, C.c_int32, C.c_int32, P, P, P]
    lib.fcm_plan.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, S, C.POINTER(S)]
    lib.fcm_launch_count.restype = C.c_uint64
    lib.fcm_status_str.argtypes = [I]
    lib.fcm_status_str.restype = C.c_char_p
    lib.fcm_last_error.restype = C.c_char_p
    for f in ("fcm_dw", "fcm_pw", "fcm_dwpw", "fcm_pwdw_r", "fcm_pwpw", "fcm_pack_pw", "fcm_plan", "fcm_version"):
        getattr(lib, f).restype = I
    _lib = lib
    return lib


def status_str(s: int) -> str:
    return load().fcm_status_str(s).decode()


def check(status: int, where: str) -> None:
    if status != FCM_OK:
        raise FcmError(status, where, load().fcm_last_error().decode())

"""FCMs on B200: Python binding of libfcm.so (include/fcm.h).

Same names as the C ABI (fcm_dw -> dw, ...). Argument marshalling only: torch supplies device
memory and the current CUDA stream; every step of the hot path runs in the library's kernels.
There is no CPU fallback -- importing the ops without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from paper_2404_19331_b200 import _lib as L

_DT = {torch.float32: L.FCM_F32, torch.bfloat16: L.FCM_BF16, torch.float16: L.FCM_F16, torch.int8: L.FCM_S8}


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _tensor(t: torch.Tensor, layout: int = L.FCM_NHWC) -> L.FcmTensor:
    if t.dtype not in _DT:
        raise TypeError(f"unsupported dtype {t.dtype}")
    if not t.is_contiguous():
        raise ValueError("tensors must be contiguous (dense NHWC / NCHW)")
    if layout == L.FCM_NHWC:
        n, h, w, c = t.shape
    else:
        n, c, h, w = t.shape
    return L.FcmTensor(t.data_ptr(), _DT[t.dtype], layout, n, h, w, c)


@dataclass
class Epilogue:
    """Conv-Norm-Act epilogue. Float: act/scale/bias (fp32 device tensors or None).
    int8: bias_q/mult_q/shift_q (int32 device tensors), zero points and clamp bounds."""
    act: int = L.ACT_NONE
    scale: Optional[torch.Tensor] = None
    bias: Optional[torch.Tensor] = None
    bias_q: Optional[torch.Tensor] = None
    mult_q: Optional[torch.Tensor] = None
    shift_q: Optional[torch.Tensor] = None
    zp_in: int = 0
    zp_out: int = 0
    qmin: int = -128
    qmax: int = 127
    residual: Optional[torch.Tensor] = None  # output-shaped shortcut added after the activation (float dtypes)

    def c(self) -> L.FcmEpilogue:
        return L.FcmEpilogue(self.act, _ptr(self.scale), _ptr(self.bias), _ptr(self.bias_q), _ptr(self.mult_q),
                             _ptr(self.shift_q), self.zp_in, self.zp_out, self.qmin, self.qmax, _ptr(self.residual))


def _geom(k: int, stride: int, pads: Optional[Sequence[int]]) -> L.FcmDwGeom:
    p = (k // 2,) * 4 if pads is None else tuple(pads)
    return L.FcmDwGeom(k, stride, *p)


def _tile(tile) -> Optional[L.FcmTile]:
    if tile is None:
        return None
    d = dict(tile)
    return L.FcmTile(d.get("tile_h", 0), d.get("tile_w", 0), d.get("tile_n", 0), d.get("c_chunk", 0),
                     d.get("n_split", 0))


def _out_hw(h, w, k, s, pads):
    pt, pl, pb, pr = (k // 2,) * 4 if pads is None else pads
    return (h + pt + pb - k) // s + 1, (w + pl + pr - k) // s + 1


def _ref(x):
    return None if x is None else C.byref(x)


def fcm_pack_pw(w_pw: torch.Tensor) -> torch.Tensor:
    """Offline PW weight packing: [C_in][C_out] -> packed (K-major [C_out][C_in])."""
    lib = L.load()
    c_in, c_out = w_pw.shape
    out = torch.empty((c_out, c_in), dtype=w_pw.dtype, device=w_pw.device)
    assert lib.fcm_pack_pw_bytes(_DT[w_pw.dtype], c_in, c_out) == out.numel() * out.element_size()
    L.check(lib.fcm_pack_pw(_DT[w_pw.dtype], c_in, c_out, _ptr(w_pw.contiguous()), _ptr(out), _stream()),
            "fcm_pack_pw")
    return out


def fcm_dw(x, w_dw, stride=1, pads=None, ep: Epilogue = Epilogue(), out=None, tile=None, layout="nhwc"):
    lib = L.load()
    k = w_dw.shape[0]
    lay = L.FCM_NHWC if layout == "nhwc" else L.FCM_NCHW
    if lay == L.FCM_NHWC:
        n, h, w, c = x.shape
    else:
        n, c, h, w = x.shape
    ho, wo = _out_hw(h, w, k, stride, pads)
    if out is None:
        shape = (n, ho, wo, c) if lay == L.FCM_NHWC else (n, c, ho, wo)
        out = torch.empty(shape, dtype=x.dtype, device=x.device)
    xt, yt, g, e, ti = _tensor(x, lay), _tensor(out, lay), _geom(k, stride, pads), ep.c(), _tile(tile)
    L.check(lib.fcm_dw(C.byref(xt), _ptr(w_dw), C.byref(g), C.byref(e), C.byref(yt), _ref(ti), _stream()), "fcm_dw")
    return out


def fcm_pw(x, w_packed, ep: Epilogue = Epilogue(), out=None, tile=None):
    lib = L.load()
    n, h, w, _ = x.shape
    if out is None:
        out = torch.empty((n, h, w, w_packed.shape[0]), dtype=x.dtype, device=x.device)
    xt, yt, e, ti = _tensor(x), _tensor(out), ep.c(), _tile(tile)
    L.check(lib.fcm_pw(C.byref(xt), _ptr(w_packed), C.byref(e), C.byref(yt), _ref(ti), _stream()), "fcm_pw")
    return out


def fcm_dwpw(x, w_dw, stride, pads, ep_dw: Epilogue, w_packed, ep_pw: Epilogue, out=None, tile=None):
    lib = L.load()
    n, h, w, _ = x.shape
    ho, wo = _out_hw(h, w, w_dw.shape[0], stride, pads)
    if out is None:
        out = torch.empty((n, ho, wo, w_packed.shape[0]), dtype=x.dtype, device=x.device)
    xt, yt, g, ed, ep, ti = _tensor(x), _tensor(out), _geom(w_dw.shape[0], stride, pads), ep_dw.c(), ep_pw.c(), \
        _tile(tile)
    L.check(lib.fcm_dwpw(C.byref(xt), _ptr(w_dw), C.byref(g), C.byref(ed), _ptr(w_packed), C.byref(ep),
                         C.byref(yt), _ref(ti), _stream()), "fcm_dwpw")
    return out


def fcm_pwpw(x, w1_packed, ep1: Epilogue, w2_packed, ep2: Epilogue, out=None, tile=None):
    """FCM PWPW: out = PW2(PW1(x)); the intermediate (w1_packed.shape[0] channels) stays on chip."""
    lib = L.load()
    n, h, w, _ = x.shape
    if out is None:
        out = torch.empty((n, h, w, w2_packed.shape[0]), dtype=x.dtype, device=x.device)
    xt, yt, e1, e2, ti = _tensor(x), _tensor(out), ep1.c(), ep2.c(), _tile(tile)
    L.check(lib.fcm_pwpw(C.byref(xt), _ptr(w1_packed), int(w1_packed.shape[0]), C.byref(e1), _ptr(w2_packed),
                         C.byref(e2), C.byref(yt), _ref(ti), _stream()), "fcm_pwpw")
    return out


def fcm_pwdw_r(x, w_packed, ep_pw: Epilogue, w_dw, stride, pads, ep_dw: Epilogue, out=None, tile=None):
    lib = L.load()
    n, h, w, _ = x.shape
    ho, wo = _out_hw(h, w, w_dw.shape[0], stride, pads)
    if out is None:
        out = torch.empty((n, ho, wo, w_packed.shape[0]), dtype=x.dtype, device=x.device)
    xt, yt, g, ep, ed, ti = _tensor(x), _tensor(out), _geom(w_dw.shape[0], stride, pads), ep_pw.c(), ep_dw.c(), \
        _tile(tile)
    L.check(lib.fcm_pwdw_r(C.byref(xt), _ptr(w_packed), C.byref(ep), _ptr(w_dw), C.byref(g), C.byref(ed),
                           C.byref(yt), _ref(ti), _stream()), "fcm_pwdw_r")
    return out


def fcm_plan(model: dict | str, gpu: dict | str | None = None) -> dict:
    """FusePlanner (host only)."""
    lib = L.load()
    mj = (model if isinstance(model, str) else json.dumps(model)).encode()
    gj = None if gpu is None else (gpu if isinstance(gpu, str) else json.dumps(gpu)).encode()
    need = C.c_size_t(0)
    cap = 1 << 16
    while True:
        buf = C.create_string_buffer(cap)
        st = lib.fcm_plan(mj, gj, buf, cap, C.byref(need))
        if st == L.FCM_E_BUFSZ and need.value > cap:
            cap = need.value
            continue
        L.check(st, "fcm_plan")
        return json.loads(buf.value.decode())


def fcm_launch_count() -> int:
    return int(L.load().fcm_launch_count())


# short aliases
dw, pw, dwpw, pwdw_r, pwpw, pack_pw, plan = fcm_dw, fcm_pw, fcm_dwpw, fcm_pwdw_r, fcm_pwpw, fcm_pack_pw, fcm_plan

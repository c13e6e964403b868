"""Value oracle: DW, PW and their fused compositions (TEST INFRASTRUCTURE -- see oracle/__init__).

Definitions (§II-B; readings R1-R12):

  DW  O[n,y,x,c]  = eps_c( sum_{i<k, j<k} X[n, y*s - pt + i, x*s - pl + j, c] * Wdw[i,j,c] )
                    out-of-image taps contribute 0 ("one filter is applied to a single channel")
                    Ho = floor((H + pt + pb - k)/s) + 1, Wo likewise
  PW  O[p,co]     = eps_co( sum_ci X[p,ci] * Wpw[ci,co] )  for every pixel p
                    ("1x1 filters span over all channels")
  eps             Conv-Norm-Activation epilogue: folded-BN scale/bias, then
                    NONE / RELU / RELU6 / SILU / GELU, then the optional residual (shortcut) add,
                    then rounding to the storage format. int8: int32 bias, fixed-point
                    requantisation, + zero point, clamp [qmin, qmax] (reading R1).
                    SILU (EfficientNet's swish) = v * sigmoid(v) = v / (1 + e^-v); GELU (CeiT / CMT)
                    = v * Phi(v) = 0.5 v (1 + erf(v / sqrt 2)); the residual is the inverted-residual
                    / MBConv / IRFFN shortcut ("inverted residual"); SURVEY §8(f) rank 4,
                    readings R4 / R24 in DESIGN.md.
  DWPW            = PW(DW(X)): the intermediate T is materialised in the feature-map dtype
                    (P:111 'fms_dt commBuffer'; P:144 int8 packed before writing ANY buffer).
  PWDW / PWDW_R   = DW(PW(X)): DW pads T, not X -- an out-of-image tap of T is the real 0
                    (int8: the zero point), never eps_pw(PW(0)) (reading R6). Recompute changes
                    cost, not value, so PWDW_R has the same oracle as PWDW.

Layout NHWC. Float tensors: float64 arrays holding exactly the stored values. int8: int64.
Accumulation in float64 (products of <=24-bit significands are exact) / exact int64.
"""
from __future__ import annotations

import numpy as np
from scipy.special import erf

from oracle.numerics import requant, round_to

ACT_NONE, ACT_RELU, ACT_RELU6, ACT_SILU, ACT_GELU = 0, 1, 2, 3, 4


def out_size(h: int, k: int, s: int, p0: int, p1: int) -> int:
    return (h + p0 + p1 - k) // s + 1


def dw_acc(x: np.ndarray, w: np.ndarray, stride: int, pads) -> np.ndarray:
    """sum_{i,j} X[n, y*s-pt+i, x*s-pl+j, c] * W[i,j,c]; X zero outside the image."""
    n, h, wd, c = x.shape
    k = w.shape[0]
    pt, pl, pb, pr = pads
    ho, wo = out_size(h, k, stride, pt, pb), out_size(wd, k, stride, pl, pr)
    xp = np.zeros((n, h + pt + pb, wd + pl + pr, c), dtype=x.dtype)
    xp[:, pt:pt + h, pl:pl + wd, :] = x
    acc = np.zeros((n, ho, wo, c), dtype=x.dtype)
    for i in range(k):
        for j in range(k):
            acc = acc + xp[:, i:i + stride * (ho - 1) + 1:stride, j:j + stride * (wo - 1) + 1:stride, :] * w[i, j, :]
    return acc


def pw_acc(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """sum_ci X[p,ci] * W[ci,co] over every pixel p (library matmul as the one step)."""
    n, h, wd, c = x.shape
    return (x.reshape(-1, c) @ w).reshape(n, h, wd, w.shape[1])


def act_float(v: np.ndarray, act: int) -> np.ndarray:
    if act == ACT_RELU:
        return np.maximum(v, 0.0)
    if act == ACT_RELU6:
        return np.minimum(np.maximum(v, 0.0), 6.0)
    if act == ACT_SILU:
        with np.errstate(over="ignore"):
            return v / (1.0 + np.exp(-v))
    if act == ACT_GELU:
        return 0.5 * v * (1.0 + erf(v / np.sqrt(2.0)))
    return v


def epilogue_float(acc: np.ndarray, p: dict, fmt: str) -> np.ndarray:
    scale = p.get("scale")
    bias = p.get("bias")
    v = acc * (1.0 if scale is None else scale) + (0.0 if bias is None else bias)
    v = act_float(v, p.get("act", ACT_NONE))
    if p.get("residual") is not None:
        v = v + p["residual"]
    return round_to(v, fmt)


def epilogue_int8(acc: np.ndarray, p: dict) -> np.ndarray:
    r = requant(acc + p["bias_q"], p["mult_q"], p["shift_q"]) + p["zp_out"]
    return np.clip(r, p["qmin"], p["qmax"])


def dw(x, w, stride, pads, p: dict, fmt: str) -> np.ndarray:
    """Layer-by-layer DW + epilogue. fmt in {'f32','bf16','f16','f64','s8'}."""
    if fmt == "s8":
        return epilogue_int8(dw_acc(np.asarray(x, np.int64) - p["zp_in"], np.asarray(w, np.int64), stride, pads), p)
    return epilogue_float(dw_acc(np.asarray(x, np.float64), np.asarray(w, np.float64), stride, pads), p, fmt)


def pw(x, w, p: dict, fmt: str) -> np.ndarray:
    if fmt == "s8":
        return epilogue_int8(pw_acc(np.asarray(x, np.int64) - p["zp_in"], np.asarray(w, np.int64)), p)
    return epilogue_float(pw_acc(np.asarray(x, np.float64), np.asarray(w, np.float64)), p, fmt)


def dwpw(x, w_dw, stride, pads, p_dw, w_pw, p_pw, fmt):
    """FCM DWPW = PW(DW(X)), T rounded to the FM dtype."""
    t = dw(x, w_dw, stride, pads, p_dw, fmt)
    return pw(t, w_pw, p_pw, fmt)


def pwdw(x, w_pw, p_pw, w_dw, stride, pads, p_dw, fmt):
    """FCM PWDW / PWDW_R = DW(PW(X)); DW zero-pads T itself (reading R6)."""
    t = pw(x, w_pw, p_pw, fmt)
    return dw(t, w_dw, stride, pads, p_dw, fmt)


def pwpw(x, w1, p1, w2, p2, fmt):
    """FCM PWPW = PW2(PW1(X)) (the paper's third FCM kind); T rounded /
    requantised to the FM dtype like every commBuffer."""
    t = pw(x, w1, p1, fmt)
    return pw(t, w2, p2, fmt)


# ----------------------------------------------------------------------------------
# magnitude bound for float tolerances (reading R10)
# ----------------------------------------------------------------------------------
def _absp(p):
    q = dict(p)
    q["scale"] = None if p.get("scale") is None else np.abs(p["scale"])
    q["bias"] = None if p.get("bias") is None else np.abs(p["bias"])
    q["act"] = ACT_NONE  # |relu(v)|, |silu(v)|, |gelu(v)| <= |v| (the latter two up to 1.13 |dv| slope)
    q["residual"] = None if p.get("residual") is None else np.abs(p["residual"])
    return q


def mag_dw(x, w, stride, pads, p):
    return dw(np.abs(x), np.abs(w), stride, pads, _absp(p), "f64")


def mag_pw(x, w, p):
    return pw(np.abs(x), np.abs(w), _absp(p), "f64")


def mag_dwpw(x, w_dw, stride, pads, p_dw, w_pw, p_pw):
    return mag_pw(mag_dw(x, w_dw, stride, pads, p_dw), w_pw, p_pw)


def mag_pwdw(x, w_pw, p_pw, w_dw, stride, pads, p_dw):
    return mag_dw(mag_pw(x, w_pw, p_pw), w_dw, stride, pads, p_dw)


def mag_pwpw(x, w1, p1, w2, p2):
    return mag_pw(mag_pw(x, w1, p1), w2, p2)

"""FusePlanner memory-access models and exact tiled counters (TEST INFRASTRUCTURE -- see oracle/__init__).

All counts are in ELEMENTS; multiply by the element size for bytes (byte width
scales every term). Symbols follow PAPER.md §IV.

Verbatim equations
  overlap   Eq. 1: (ceil(CW/TW)-1)(FW-S)CH + (ceil(CH/TH)-1)(FH-S)CW,
            each (F-S) clamped at 0; TileW/TileH are IFM-space tile dims (reading R16).
  pw_gma    Eq. 2: ceil(W/WT)*IFM + OFM + ceil(OFM/OFMT)*W
  dw_gma    Eq. 3: 2*D*Overlap + IFM + OFM + ceil(OFM_HW/OFMT_HW)*W
  pwdw_gma  Eq. 4: (2*PwD*DwOverlap + PwIFM) * max(ceil(PwW/PwWT), ceil(DwW/DwWT))
                               + ceil(DwOFM/DwOFMT)*PwW + ceil(DwOFM_HW/DwOFMT_HW)*DwW
            'paper' mode prints no final store term; 'consistent' adds DwOFM (reading R15).
  dwpw_gma  constructed "similarly" -- not printed in the paper (reading R13):
            (2*DwD*DwOverlap + DwIFM)*ceil(PwW/PwWT) + ceil(PwOFM_HW/PwOFMT_HW)*ceil(PwW/PwWT)*DwW
            + ceil(PwOFM/PwOFMT)*PwW + PwOFM

Exact counters (reading R13/R14): an OS-LWS execution is a set of work units, one
per (output spatial tile) x (weight partition). A unit loads every DISTINCT input element
its outputs need (halo clipped at the image edge; padding is never fetched), its weight
partition, and stores its outputs once. The counter sums those per-unit counts.

Decision rule: fuse iff min FCM GMA < sum of its layers' min LBL GMA (strict).
"""
from __future__ import annotations

from math import ceil


# ------------------------------------------------------------------ verbatim equations
def overlap(ch: int, cw: int, th: int, tw: int, fh: int, fw: int, s: int) -> int:
    """Eq. 1."""
    return (ceil(cw / tw) - 1) * max(fw - s, 0) * ch + (ceil(ch / th) - 1) * max(fh - s, 0) * cw


def pw_gma(ifm: int, ofm: int, w: int, wt: int, ofmt: int) -> int:
    """Eq. 2."""
    return ceil(w / wt) * ifm + ofm + ceil(ofm / ofmt) * w


def dw_gma(d: int, ovl: int, ifm: int, ofm: int, ofm_hw: int, ofmt_hw: int, w: int) -> int:
    """Eq. 3."""
    return 2 * d * ovl + ifm + ofm + ceil(ofm_hw / ofmt_hw) * w


def pwdw_gma(pw_d, dw_ovl, pw_ifm, pw_w, pw_wt, dw_w, dw_wt, dw_ofm, dw_ofmt, dw_ofm_hw, dw_ofmt_hw,
             mode="consistent") -> int:
    """Eq. 4 (PWDW / PWDW_R)."""
    g = (2 * pw_d * dw_ovl + pw_ifm) * max(ceil(pw_w / pw_wt), ceil(dw_w / dw_wt)) \
        + ceil(dw_ofm / dw_ofmt) * pw_w + ceil(dw_ofm_hw / dw_ofmt_hw) * dw_w
    return g + (dw_ofm if mode == "consistent" else 0)


def dwpw_gma(dw_d, dw_ovl, dw_ifm, dw_w, pw_w, pw_wt, pw_ofm, pw_ofmt, pw_ofm_hw, pw_ofmt_hw) -> int:
    """DWPW by the construction rule of P:211 (reading R13)."""
    nw = ceil(pw_w / pw_wt)
    return (2 * dw_d * dw_ovl + dw_ifm) * nw + ceil(pw_ofm_hw / pw_ofmt_hw) * nw * dw_w \
        + ceil(pw_ofm / pw_ofmt) * pw_w + pw_ofm


def fused_wins(fcm_min: int, lbl_sum: int) -> bool:
    """fuse when the FCM estimate is LESS THAN the LBL estimates of its layers."""
    return fcm_min < lbl_sum


# ------------------------------------------------------------------ exact counters
def tiles_1d(n: int, t: int):
    """Output tile ranges [a, b) of extent t covering 0..n-1 (last tile ragged)."""
    return [(a, min(a + t, n)) for a in range(0, n, t)]


def touched(a: int, b: int, k: int, s: int, p: int, n_in: int) -> int:
    """Number of distinct in-image input rows read by output rows [a, b): {y*s-p+i}, i<k."""
    return len({y * s - p + i for y in range(a, b) for i in range(k)} & set(range(n_in)))


def dw_exact(h, w, c, k, s, pads, th, tw, td):
    """Exact DW counts: units = spatial tile x channel slice. Returns dict of element counts."""
    pt, pl, pb, pr = pads
    ho, wo = (h + pt + pb - k) // s + 1, (w + pl + pr - k) // s + 1
    ifm = wts = 0
    for (y0, y1) in tiles_1d(ho, th):
        ny = touched(y0, y1, k, s, pt, h)
        for (x0, x1) in tiles_1d(wo, tw):
            nx = touched(x0, x1, k, s, pl, w)
            for (c0, c1) in tiles_1d(c, td):
                ifm += ny * nx * (c1 - c0)
                wts += k * k * (c1 - c0)
    return {"ifm": ifm, "w": wts, "ofm": ho * wo * c, "total": ifm + wts + ho * wo * c}


def pw_exact(h, w, c_in, c_out, th, tw, wt_filters):
    """Exact PW counts, OS-LWS: unit = spatial tile x weight partition (wt_filters filters)."""
    ifm = wts = 0
    for (y0, y1) in tiles_1d(h, th):
        for (x0, x1) in tiles_1d(w, tw):
            for (f0, f1) in tiles_1d(c_out, wt_filters):
                ifm += (y1 - y0) * (x1 - x0) * c_in
                wts += c_in * (f1 - f0)
    return {"ifm": ifm, "w": wts, "ofm": h * w * c_out, "total": ifm + wts + h * w * c_out}


def dwpw_exact(h, w, c_in, c_out, k, s, pads, th, tw, n_cta):
    """Exact fused DWPW counts: unit = output spatial tile x C_out slice; every unit re-reads the
    X halo over ALL C_in channels (the intermediate must contain all channels) and the
    DW weights, plus its PW weight slice."""
    pt, pl, pb, pr = pads
    ho, wo = (h + pt + pb - k) // s + 1, (w + pl + pr - k) // s + 1
    ifm = wts = 0
    for (y0, y1) in tiles_1d(ho, th):
        ny = touched(y0, y1, k, s, pt, h)
        for (x0, x1) in tiles_1d(wo, tw):
            nx = touched(x0, x1, k, s, pl, w)
            for (f0, f1) in tiles_1d(c_out, n_cta):
                ifm += ny * nx * c_in
                wts += k * k * c_in + c_in * (f1 - f0)
    ofm = ho * wo * c_out
    return {"ifm": ifm, "w": wts, "ofm": ofm, "total": ifm + wts + ofm, "redundant_macs": 0}


def pwdw_exact(h, w, c_in, c_mid, k, s, pads, th, tw, td):
    """Exact fused PWDW(_R) counts: unit = DW output tile x intermediate-channel slice td.
    The unit computes T over its (clipped) DW halo tile: loads X there over all C_in, the PW
    weights of its slice and the DW weights of its slice; recomputed T pixels are redundant."""
    pt, pl, pb, pr = pads
    ho, wo = (h + pt + pb - k) // s + 1, (w + pl + pr - k) // s + 1
    ifm = wts = halo_px = 0
    for (y0, y1) in tiles_1d(ho, th):
        ny = touched(y0, y1, k, s, pt, h)
        for (x0, x1) in tiles_1d(wo, tw):
            nx = touched(x0, x1, k, s, pl, w)
            for (c0, c1) in tiles_1d(c_mid, td):
                px = ny * nx
                ifm += px * c_in
                wts += c_in * (c1 - c0) + k * k * (c1 - c0)
                halo_px += px * (c1 - c0)
    ofm = ho * wo * c_mid
    redundant = (halo_px - h * w * c_mid) * c_in
    return {"ifm": ifm, "w": wts, "ofm": ofm, "total": ifm + wts + ofm, "redundant_macs": redundant}


def redundancy_ratio(h, w, c_in, c_mid, k, s, pads, th, tw, td):
    """Table 2 semantics: redundant MACs / (PW MACs + DW MACs + redundant MACs)."""
    e = pwdw_exact(h, w, c_in, c_mid, k, s, pads, th, tw, td)
    pt, pl, pb, pr = pads
    ho, wo = (h + pt + pb - k) // s + 1, (w + pl + pr - k) // s + 1
    pw_macs = h * w * c_in * c_mid
    dw_macs = ho * wo * c_mid * k * k
    r = e["redundant_macs"]
    return r / (pw_macs + dw_macs + r)


def compulsory(kind: str, n, h, w, c_in, c_out, k=1, s=1, c_mid=None):
    """Compulsory HBM elements per launch: activations per image x n, weights once.
    kind: 'dw' | 'pw' | 'dwpw' | 'pwdw'. For dw, c_out == c_in; for pwdw c_out is C_mid."""
    p = k // 2
    ho, wo = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    if kind == "dw":
        return n * (h * w * c_in + ho * wo * c_in) + k * k * c_in
    if kind == "pw":
        return n * h * w * (c_in + c_out) + c_in * c_out
    if kind == "dwpw":
        return n * (h * w * c_in + ho * wo * c_out) + k * k * c_in + c_in * c_out
    if kind == "pwdw":
        return n * (h * w * c_in + ho * wo * c_out) + c_in * c_out + k * k * c_out
    raise ValueError(kind)

"""Seeded parity cases shared by the GPU tests and __graft_entry__.smoke() (test infrastructure).

A case builds inputs with synth (same stored bits on both sides), runs the oracle on CPU and
the CUDA path through the C ABI, and compares:
  int8   bit-exact
  float  |gpu - oracle| <= rtol * mag + 1e-30, mag = the layer chain on |X|, |W|, |scale|,
         |bias| (reading R10); rtol = 1e-5 (fp32) / 2e-2 (bf16, fp16) from north_star.
"""
from __future__ import annotations

import numpy as np
import torch

import synth
from oracle import conv as oc

DT = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16, "s8": torch.int8}
RTOL = {"f32": 1e-5, "bf16": 2e-2, "f16": 2e-2}


def stored(a: np.ndarray, fmt: str) -> torch.Tensor:
    """Cast generated values to the storage dtype (CPU tensor)."""
    if fmt == "s8":
        return torch.from_numpy(np.asarray(a, dtype=np.int64)).to(torch.int8)
    return torch.from_numpy(np.asarray(a, dtype=np.float64)).to(DT[fmt])


def as_np(t: torch.Tensor, fmt: str) -> np.ndarray:
    t = t.detach().cpu()
    return t.to(torch.int64).numpy() if fmt == "s8" else t.to(torch.float64).numpy()


def layer_params(seed, name, kind, fmt, c_in, c_out=None, k=3, act=synth.ACT_RELU6, zp_out=0):
    """Host-side params (numpy, exact stored values) for one layer."""
    if fmt == "s8":
        if kind == "dw":
            p = synth.int8_dw_params(seed, name, k, c_in, act)
        else:
            p = synth.int8_pw_params(seed, name, c_in, c_out, act)
        p["zp_out"] = zp_out
        if act != synth.ACT_NONE:
            p["qmin"] = zp_out
        return p
    if kind == "dw":
        p = synth.float_dw_params(seed, name, k, c_in, act)
    else:
        p = synth.float_pw_params(seed, name, c_in, c_out, act)
    p["w"] = as_np(stored(p["w"], fmt), fmt)
    p["scale"] = p["scale"].astype(np.float32).astype(np.float64)
    p["bias"] = p["bias"].astype(np.float32).astype(np.float64)
    return p


def device_epi(p, fmt, dev, residual=None):
    import paper_2404_19331_b200 as fcm
    if fmt == "s8":
        i32 = lambda a: torch.as_tensor(np.asarray(a), dtype=torch.int32, device=dev)
        return fcm.Epilogue(act=p.get("act", 0), bias_q=i32(p["bias_q"]), mult_q=i32(p["mult_q"]),
                            shift_q=i32(p["shift_q"]), zp_in=p.get("zp_in", 0), zp_out=p.get("zp_out", 0),
                            qmin=p["qmin"], qmax=p["qmax"])
    f32 = lambda a: torch.as_tensor(np.asarray(a), dtype=torch.float32, device=dev)
    return fcm.Epilogue(act=p["act"], scale=f32(p["scale"]), bias=f32(p["bias"]), residual=residual)


def make_x(seed, fmt, n, h, w, c, role="x"):
    kind = "int8" if fmt == "s8" else "float"
    return stored(synth.activations(seed, role, 0, n, h, w, c, kind), fmt)


def compare(gpu: np.ndarray, ref: np.ndarray, mag, fmt: str, what: str):
    assert gpu.shape == ref.shape, (what, gpu.shape, ref.shape)
    if fmt == "s8":
        bad = np.argwhere(gpu != ref)
        assert bad.size == 0, f"{what}: {len(bad)} int8 mismatches, first at {bad[0].tolist()}: " \
                              f"gpu {gpu[tuple(bad[0])]} oracle {ref[tuple(bad[0])]}"
        return 0.0
    err = np.abs(gpu - ref)
    bound = RTOL[fmt] * mag + 1e-30
    bad = np.argwhere(err > bound)
    assert bad.size == 0, f"{what}: {len(bad)} elements outside tolerance; first {bad[0].tolist()}: gpu " \
                          f"{gpu[tuple(bad[0])]} oracle {ref[tuple(bad[0])]} mag {mag[tuple(bad[0])]}"
    return float((err / np.maximum(mag, 1e-30)).max())


class Case:
    """One fused or unfused layer on seeded inputs, both sides."""

    def __init__(self, op, fmt, n, h, w, c_in, c_out=None, k=3, s=1, pads=None, seed=synth.SEED, tile=None,
                 act_dw=synth.ACT_RELU6, act_pw=synth.ACT_NONE, c_mid=None, residual=False):
        self.op, self.fmt, self.k, self.s, self.tile = op, fmt, k, s, tile
        self.pads = (k // 2,) * 4 if pads is None else tuple(pads)
        self.x = make_x(seed, fmt, n, h, w, c_in)
        self.c_in, self.c_out = c_in, c_out
        self.res = None  # residual (shortcut) tensor of the output's shape, SURVEY §8(f) rank 4
        if residual:
            pt, pl, pb, pr = self.pads
            ho = oc.out_size(h, k, s, pt, pb) if op == "dwpw" else h
            wo = oc.out_size(w, k, s, pl, pr) if op == "dwpw" else w
            self.res = make_x(seed, fmt, n, ho, wo, c_out, role="residual")
        if op in ("dw",):
            self.pd = layer_params(seed, "dw", "dw", fmt, c_in, k=k, act=act_dw)
        elif op == "pw":
            self.pp = layer_params(seed, "pw", "pw", fmt, c_in, c_out, act=act_pw)
        elif op == "dwpw":
            self.pd = layer_params(seed, "dw", "dw", fmt, c_in, k=k, act=act_dw)
            self.pp = layer_params(seed, "pw", "pw", fmt, c_in, c_out, act=act_pw)
        elif op == "pwdw":
            self.pp = layer_params(seed, "pw", "pw", fmt, c_in, c_out, act=synth.ACT_RELU6)
            self.pd = layer_params(seed, "dw", "dw", fmt, c_out, k=k, act=act_dw)
        elif op == "pwpw":
            self.c_mid = c_mid
            self.pp1 = layer_params(seed, "pw1", "pw", fmt, c_in, c_mid, act=act_dw)
            self.pp2 = layer_params(seed, "pw2", "pw", fmt, c_mid, c_out, act=act_pw)
        else:
            raise ValueError(op)
        if self.res is not None:
            (self.pp2 if op == "pwpw" else self.pp)["residual"] = as_np(self.res, fmt)

    # ------------------------------------------------------------------ oracle
    def oracle(self):
        x = as_np(self.x, self.fmt)
        f = self.fmt
        if self.op == "dw":
            ref = oc.dw(x, self.pd["w"], self.s, self.pads, self.pd, f)
            mag = None if f == "s8" else oc.mag_dw(x, self.pd["w"], self.s, self.pads, self.pd)
        elif self.op == "pw":
            ref = oc.pw(x, self.pp["w"], self.pp, f)
            mag = None if f == "s8" else oc.mag_pw(x, self.pp["w"], self.pp)
        elif self.op == "dwpw":
            ref = oc.dwpw(x, self.pd["w"], self.s, self.pads, self.pd, self.pp["w"], self.pp, f)
            mag = None if f == "s8" else oc.mag_dwpw(x, self.pd["w"], self.s, self.pads, self.pd, self.pp["w"],
                                                     self.pp)
        elif self.op == "pwpw":
            ref = oc.pwpw(x, self.pp1["w"], self.pp1, self.pp2["w"], self.pp2, f)
            mag = None if f == "s8" else oc.mag_pwpw(x, self.pp1["w"], self.pp1, self.pp2["w"], self.pp2)
        else:
            ref = oc.pwdw(x, self.pp["w"], self.pp, self.pd["w"], self.s, self.pads, self.pd, f)
            mag = None if f == "s8" else oc.mag_pwdw(x, self.pp["w"], self.pp, self.pd["w"], self.s, self.pads,
                                                     self.pd)
        return ref, mag

    # ------------------------------------------------------------------ CUDA path (C ABI)
    def gpu(self, dev="cuda:0"):
        import paper_2404_19331_b200 as fcm
        f = self.fmt
        x = self.x.to(dev)
        if hasattr(self, "pd"):
            wdw = stored(self.pd["w"], f).to(dev)
            ed = device_epi(self.pd, f, dev)
        res = None if self.res is None else self.res.to(dev)
        if hasattr(self, "pp"):
            wpk = fcm.pack_pw(stored(self.pp["w"], f).to(dev))
            ep = device_epi(self.pp, f, dev, res)
        if self.op == "pwpw":
            w1 = fcm.pack_pw(stored(self.pp1["w"], f).to(dev))
            w2 = fcm.pack_pw(stored(self.pp2["w"], f).to(dev))
            y = fcm.pwpw(x, w1, device_epi(self.pp1, f, dev), w2, device_epi(self.pp2, f, dev, res))
        elif self.op == "dw":
            y = fcm.dw(x, wdw, self.s, self.pads, ed, tile=self.tile)
        elif self.op == "pw":
            y = fcm.pw(x, wpk, ep, tile=self.tile)
        elif self.op == "dwpw":
            y = fcm.dwpw(x, wdw, self.s, self.pads, ed, wpk, ep, tile=self.tile)
        else:
            y = fcm.pwdw_r(x, wpk, ep, wdw, self.s, self.pads, ed, tile=self.tile)
        torch.cuda.synchronize()
        return as_np(y, f)

    def check(self, dev="cuda:0"):
        ref, mag = self.oracle()
        return compare(self.gpu(dev), ref, mag, self.fmt, f"{self.op}/{self.fmt}")


def oracle_entry(e, layers, prm, x, fmt, res=None):
    """Oracle output (and R10 magnitude, None for int8) of one plan entry applied to input x;
    res = the shortcut tensor its output epilogue adds, or None."""
    op, lids = e["op"], e["layers"]
    if res is not None:
        prm = dict(prm)
        prm[lids[-1]] = dict(prm[lids[-1]], residual=res)
    pads = lambda l: (l["k"] // 2,) * 4
    f64 = fmt != "s8"
    if op == "dw":
        l, p = layers[lids[0]], prm[lids[0]]
        ref = oc.dw(x, p["w"], l["stride"], pads(l), p, fmt)
        return ref, (oc.mag_dw(x, p["w"], l["stride"], pads(l), p) if f64 else None)
    if op == "pw":
        p = prm[lids[0]]
        return oc.pw(x, p["w"], p, fmt), (oc.mag_pw(x, p["w"], p) if f64 else None)
    if op == "dwpw":
        l, pd, pp = layers[lids[0]], prm[lids[0]], prm[lids[1]]
        ref = oc.dwpw(x, pd["w"], l["stride"], pads(l), pd, pp["w"], pp, fmt)
        return ref, (oc.mag_dwpw(x, pd["w"], l["stride"], pads(l), pd, pp["w"], pp) if f64 else None)
    if op == "pwdw_r":
        l, pp, pd = layers[lids[1]], prm[lids[0]], prm[lids[1]]
        ref = oc.pwdw(x, pp["w"], pp, pd["w"], l["stride"], pads(l), pd, fmt)
        return ref, (oc.mag_pwdw(x, pp["w"], pp, pd["w"], l["stride"], pads(l), pd) if f64 else None)
    if op == "pwpw":
        p1, p2 = prm[lids[0]], prm[lids[1]]
        return oc.pwpw(x, p1["w"], p1, p2["w"], p2, fmt), (oc.mag_pwpw(x, p1["w"], p1, p2["w"], p2) if f64 else None)
    raise ValueError(op)

"""Whole-stack oracle: a network's DW/PW layers evaluated one by one with oracle.conv
(TEST INFRASTRUCTURE -- see oracle/__init__).

The unfused composition is the reference for any plan: an FCM computes exactly PW(DW(X)) or
DW(PW(X)) with the intermediate rounded to the feature-map dtype, so the
fused and unfused stacks have the same oracle. Inputs and parameters come from synth (the same
seeded generators the GPU path uses), cast to the storage dtype by torch (input recipe).
"""
from __future__ import annotations

import numpy as np
import torch

import synth
from oracle import conv
from synth.networks import NETWORKS, block_source, layer_ids, network_params

_TD = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}


def _stored(a, dtype):
    if dtype == "s8":
        return np.asarray(a, dtype=np.int64)
    return torch.from_numpy(np.asarray(a, dtype=np.float64)).to(_TD[dtype]).to(torch.float64).numpy()


def _images(net, dtype, role, n0, n, h, w, c, seed):
    kind = "int8" if dtype == "s8" else "float"
    return _stored(synth.activations(seed, role, n0, n, h, w, c, kind), dtype)


def params(net, dtype, seed=synth.SEED):
    """Parameters as the GPU stores them: weights in the storage dtype, float scale/bias in fp32."""
    out = {}
    for lid, p in network_params(seed, net, dtype).items():
        q = dict(p)
        q["w"] = _stored(p["w"], dtype)
        if dtype != "s8":
            q["scale"] = p["scale"].astype(np.float32).astype(np.float64)
            q["bias"] = p["bias"].astype(np.float32).astype(np.float64)
        out[lid] = q
    return out


def forward(net, dtype, n0, n, seed=synth.SEED, prm=None, keep=False):
    """Run images [n0, n0+n) through the whole stack. Returns the final output (NHWC), or with
    keep=True a dict layer_id -> output."""
    blocks = NETWORKS[net]()
    prm = prm or params(net, dtype, seed)
    ids = layer_ids(blocks)
    first = ids[0][2]
    c0 = first["c"] if first["kind"] == "dw" else first["c_in"]
    x0 = _images(net, dtype, f"{net}/input", n0, n, first["h"], first["w"], c0, seed)
    cur, outs, stage, inputs = x0, {}, {}, {}
    for lid, bi, l in ids:
        if lid.endswith(".0"):
            kind, role = block_source(net, blocks, bi)
            if kind == "stage":
                c = l["c"] if l["kind"] == "dw" else l["c_in"]
                if role not in stage:
                    stage[role] = x0 if bi == 0 else _images(net, dtype, role, n0, n, l["h"], l["w"], c, seed)
                cur = stage[role]
        inputs[lid] = cur
        p = prm[lid]
        if l.get("residual_from") is not None and dtype != "s8":  # shortcut (float only)
            p = dict(p, residual=inputs[l["residual_from"]])
        if l["kind"] == "dw":
            k = l["k"]
            cur = conv.dw(cur, p["w"], l["stride"], (k // 2,) * 4, p, dtype)
        else:
            cur = conv.pw(cur, p["w"], p, dtype)
        if keep:
            outs[lid] = cur
    return outs if keep else cur

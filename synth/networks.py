"""DW/PW layer tables of the BASELINE networks (public architectures).

Only shapes: no arithmetic of the method. Each network is a list of *blocks*; a block is
a list of layer dicts in execution order:

  {"kind": "dw", "h", "w", "c", "k", "stride", "act"}      (pads are k//2 on all sides)
  {"kind": "pw", "h", "w", "c_in", "c_out", "act"}

Stem convolutions, SE, pooling and classifier heads are not DW/PW layers and are omitted
(SURVEY §8(f) rank 4); residual adds are likewise outside the paper's model.
"""
from __future__ import annotations

from synth import ACT_NONE, ACT_RELU6


def _dw(h, w, c, k, s, act=ACT_RELU6):
    return {"kind": "dw", "h": h, "w": w, "c": c, "k": k, "stride": s, "act": act}


def _pw(h, w, ci, co, act=ACT_RELU6):
    return {"kind": "pw", "h": h, "w": w, "c_in": ci, "c_out": co, "act": act}


def single_dwpw():
    """configs[0]: IFM 1x16x14x14 (NCHW in BASELINE, NHWC here), DW 3x3 s1 p1, PW 16->32."""
    return [[_dw(14, 14, 16, 3, 1), _pw(14, 14, 16, 32, ACT_NONE)]]


def mobilenet_v1():
    """configs[1]: 13 DSC blocks of MobileNetV1 at 224x224 (after the 3x3 s2 stem)."""
    spec = [(112, 32, 64, 1), (112, 64, 128, 2), (56, 128, 128, 1), (56, 128, 256, 2),
            (28, 256, 256, 1), (28, 256, 512, 2)] + [(14, 512, 512, 1)] * 5 + \
           [(14, 512, 1024, 2), (7, 1024, 1024, 1)]
    blocks = []
    for hw, ci, co, s in spec:
        ho = hw // s
        blocks.append([_dw(hw, hw, ci, 3, s), _pw(ho, ho, ci, co)])
    return blocks


def _inverted_residuals(table, k_of=None):
    """table rows: (t, c_out, n, s[, k]); input 112x112x32."""
    blocks, hw, c = [], 112, 32
    for row in table:
        t, co, n, s = row[:4]
        k = row[4] if len(row) > 4 else 3
        for i in range(n):
            st = s if i == 0 else 1
            ho = hw // st
            b = []
            mid = c * t
            if t != 1:
                b.append(_pw(hw, hw, c, mid))
            b.append(_dw(hw, hw, mid, k, st))
            b.append(_pw(ho, ho, mid, co, ACT_NONE))
            blocks.append(b)
            hw, c = ho, co
    return blocks, hw, c


def mobilenet_v2():
    """configs[2]: 17 inverted residuals (t=6 except block 0) + final PW 320->1280."""
    blocks, hw, c = _inverted_residuals([(1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2),
                                         (6, 96, 3, 1), (6, 160, 3, 2), (6, 320, 1, 1)])
    blocks.append([_pw(hw, hw, c, 1280)])
    return blocks


def efficientnet_b0():
    """configs[3]: 16 MBConv blocks (3x3 and 5x5 DW, SE omitted, RELU6) + final PW 320->1280."""
    blocks, hw, c = _inverted_residuals([(1, 16, 1, 1, 3), (6, 24, 2, 2, 3), (6, 40, 2, 2, 5),
                                         (6, 80, 3, 2, 3), (6, 112, 3, 1, 5), (6, 192, 4, 2, 5),
                                         (6, 320, 1, 1, 3)])
    blocks.append([_pw(hw, hw, c, 1280)])
    return blocks


def cvt13_projections():
    """configs[4]: CvT-13 Q (DW3 s1 + PW) and K, V (DW3 s2 + PW) projections, BN, no activation."""
    blocks = []
    for hw, c, nblk in [(56, 64, 1), (28, 192, 2), (14, 384, 10)]:
        for _ in range(nblk):
            blocks.append([_dw(hw, hw, c, 3, 1, ACT_NONE), _pw(hw, hw, c, c, ACT_NONE)])  # Q
            for _kv in range(2):
                blocks.append([_dw(hw, hw, c, 3, 2, ACT_NONE), _pw(hw // 2, hw // 2, c, c, ACT_NONE)])
    return blocks


NETWORKS = {
    "single_dwpw": single_dwpw,
    "mobilenet_v1": mobilenet_v1,
    "mobilenet_v2": mobilenet_v2,
    "efficientnet_b0": efficientnet_b0,
    "cvt13": cvt13_projections,
}


def layer_ids(blocks):
    """[(id, block index, layer dict)] in execution order; ids are 'b<block>.<i>'."""
    return [(f"b{bi}.{li}", bi, l) for bi, b in enumerate(blocks) for li, l in enumerate(b)]


def network_params(seed: int, net: str, dtype: str) -> dict:
    """Per-layer synthetic parameters of a network (numpy; weights NOT yet cast to the storage
    dtype). int8 requantisers assume sigma_in = 73.9 for the first layer and 32 afterwards."""
    import synth
    out = {}
    sigma = 73.9
    for lid, _, l in layer_ids(NETWORKS[net]()):
        name = f"{net}/{lid}"
        if dtype == "s8":
            if l["kind"] == "dw":
                p = synth.int8_dw_params(seed, name, l["k"], l["c"], l["act"], sigma)
            else:
                p = synth.int8_pw_params(seed, name, l["c_in"], l["c_out"], l["act"], sigma)
            sigma = 32.0
        else:
            if l["kind"] == "dw":
                p = synth.float_dw_params(seed, name, l["k"], l["c"], l["act"])
            else:
                p = synth.float_pw_params(seed, name, l["c_in"], l["c_out"], l["act"])
        out[lid] = p
    return out


def block_source(net: str, blocks, bi: int):
    """Where block bi reads its input: ('chain', None) = previous block's output, or
    ('stage', role) = a stage token map shared by all CvT projections of that stage."""
    if net != "cvt13":
        return ("chain", None)
    l = blocks[bi][0]
    return ("stage", f"{net}/stage_{l['h']}x{l['c']}")

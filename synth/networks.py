"""DW/PW layer tables of the BASELINE networks (public architectures).

Only shapes: no arithmetic of the method. Each network is a list of *blocks*; a block is
a list of layer dicts in execution order:

  {"kind": "dw", "h", "w", "c", "k", "stride", "act"}      (pads are k//2 on all sides)
  {"kind": "pw", "h", "w", "c_in", "c_out", "act"[, "residual_from": layer id]}

"residual_from" (the inverted-residual shortcut of P:50): the PW's epilogue
adds the INPUT of that layer (same shape as the PW's output) after its activation -- MobileNetV2 /
EfficientNet-B0 / ProxylessNAS blocks with stride 1 and C_in == C_out, CeiT's LeFF and CMT's
IRFFN (x + FFN(x)), Xception's middle-flow blocks. Stem convolutions, SE, pooling and classifier
heads are not DW/PW layers and are omitted; so are shortcuts that are not identities (Xception's
1x1 s2 projections) and CMT's DW-local shortcut (reading R24).
"""
from __future__ import annotations

from synth import ACT_GELU, ACT_NONE, ACT_RELU, ACT_RELU6, ACT_SILU


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


def _inverted_residuals(table, act=ACT_RELU6, bi0=0):
    """table rows: (t, c_out, n, s[, k]); input 112x112x32. A block with stride 1 and
    C_in == C_out adds its input to the projection output (residual_from its first layer)."""
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
                b.append(_pw(hw, hw, c, mid, act))
            b.append(_dw(hw, hw, mid, k, st, act))
            b.append(_pw(ho, ho, mid, co, ACT_NONE))
            if st == 1 and c == co:
                b[-1]["residual_from"] = f"b{bi0 + len(blocks)}.0"
            blocks.append(b)
            hw, c = ho, co
    return blocks, hw, c


def mobilenet_v2():
    """configs[2]: 17 inverted residuals (t=6 except block 0; 10 with the identity shortcut) +
    final PW 320->1280."""
    blocks, hw, c = _inverted_residuals([(1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2),
                                         (6, 96, 3, 1), (6, 160, 3, 2), (6, 320, 1, 1)])
    blocks.append([_pw(hw, hw, c, 1280)])
    return blocks


def efficientnet_b0():
    """configs[3]: 16 MBConv blocks (3x3 and 5x5 DW, SiLU, identity shortcuts; SE omitted) +
    final PW 320->1280 (SiLU)."""
    blocks, hw, c = _inverted_residuals([(1, 16, 1, 1, 3), (6, 24, 2, 2, 3), (6, 40, 2, 2, 5),
                                         (6, 80, 3, 2, 3), (6, 112, 3, 1, 5), (6, 192, 4, 2, 5),
                                         (6, 320, 1, 1, 3)], act=ACT_SILU)
    blocks.append([_pw(hw, hw, c, 1280, ACT_SILU)])
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


def proxylessnas_gpu():
    """the MBConv DW/PW layers of ProxylessNAS-GPU
    (3x3 / 5x5 / 7x7 DW, expansions 1 / 3 / 6) after the 3x3 s2 stem (112x112x40), + final
    PW 432->1728. Per-block (expansion, kernel) choices follow the published GPU architecture as
    recalled without network access (reading R23); SE-free, RELU6."""
    spec = [(1, 24, 1, 3), (3, 32, 2, 5), (3, 32, 1, 3), (3, 56, 2, 7), (3, 56, 1, 3), (6, 112, 2, 7),
            (3, 112, 1, 5), (6, 128, 1, 5), (3, 128, 1, 3), (3, 128, 1, 5), (6, 256, 2, 7), (6, 256, 1, 7),
            (6, 256, 1, 7), (6, 256, 1, 5), (6, 432, 1, 7)]
    blocks, hw, c = [], 112, 40
    for t, co, st, k in spec:
        ho = hw // st
        b = []
        if t != 1:
            b.append(_pw(hw, hw, c, c * t))
        b.append(_dw(hw, hw, c * t, k, st))
        b.append(_pw(ho, ho, c * t, co, ACT_NONE))
        if st == 1 and c == co:
            b[-1]["residual_from"] = f"b{len(blocks)}.0"
        blocks.append(b)
        hw, c = ho, co
    blocks.append([_pw(hw, hw, c, 1728)])
    return blocks


def xception():
    """the separable convolutions of Xception at 299x299
    (entry flow after the two stem convs, 8x3 middle flow, exit flow). A separable conv is
    DW 3x3 (no BN/activation in between) -> PW, BN, ReLU. Max-pools between entry/exit blocks and
    the 1x1 s2 residual shortcuts are not DW/PW layers (omitted); a block after a pool reads a
    fresh map of the pooled size. Each middle-flow module (3 separable convs) adds its input to
    its output (identity shortcut: residual_from the first DW of the module)."""
    spec = [(147, 64, 128), (147, 128, 128), (74, 128, 256), (74, 256, 256), (37, 256, 728), (37, 728, 728)]
    spec += [(19, 728, 728)] * 24 + [(19, 728, 728), (19, 728, 1024), (10, 1024, 1536), (10, 1536, 2048)]
    blocks = [[_dw(hw, hw, ci, 3, 1, ACT_NONE), _pw(hw, hw, ci, co, ACT_RELU)] for hw, ci, co in spec]
    for m in range(8):  # middle flow: blocks 6 + 3m .. 8 + 3m
        blocks[8 + 3 * m][-1]["residual_from"] = f"b{6 + 3 * m}.0"
    return blocks


def ceit_leff():
    """the LeFF modules of CeiT-T (12 blocks on the 14x14
    token map, C = 192, expansion 4): PW 192->768 + GELU, DW 3x3 + GELU, PW 768->192, + the
    block's shortcut x + LeFF(x); attention sits between blocks, so each LeFF reads the stage map."""
    blocks = []
    for i in range(12):
        b = [_pw(14, 14, 192, 768, ACT_GELU), _dw(14, 14, 768, 3, 1, ACT_GELU), _pw(14, 14, 768, 192, ACT_NONE)]
        b[-1]["residual_from"] = f"b{i}.0"
        blocks.append(b)
    return blocks


def cmt_irffn():
    """the IRFFN modules of CMT-S (stages 56/28/14/7 with
    C = 64/128/256/512 and 3/3/16/3 blocks, expansion 4): PW C->4C + GELU, DW 3x3 + GELU, PW 4C->C,
    + the block's shortcut x + IRFFN(x). The DW-local shortcut inside IRFFN is omitted (a DW
    epilogue residual, reading R24); each IRFFN reads its stage map."""
    blocks = []
    for hw, c, n in [(56, 64, 3), (28, 128, 3), (14, 256, 16), (7, 512, 3)]:
        for _ in range(n):
            b = [_pw(hw, hw, c, 4 * c, ACT_GELU), _dw(hw, hw, 4 * c, 3, 1, ACT_GELU), _pw(hw, hw, 4 * c, c, ACT_NONE)]
            b[-1]["residual_from"] = f"b{len(blocks)}.0"
            blocks.append(b)
    return blocks


NETWORKS = {
    "single_dwpw": single_dwpw,
    "mobilenet_v1": mobilenet_v1,
    "mobilenet_v2": mobilenet_v2,
    "efficientnet_b0": efficientnet_b0,
    "cvt13": cvt13_projections,
    "xception": xception,
    "proxylessnas_gpu": proxylessnas_gpu,
    "ceit_leff": ceit_leff,
    "cmt_irffn": cmt_irffn,
}

# networks whose DW/PW blocks are separated by non-DW/PW layers (attention): every block reads
# the stage's token map instead of the previous block's output
_STAGE_FED = {"cvt13", "ceit_leff", "cmt_irffn"}


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
    l = blocks[bi][0]
    c = l["c"] if l["kind"] == "dw" else l["c_in"]
    if net in _STAGE_FED:
        return ("stage", f"{net}/stage_{l['h']}x{c}")
    if bi == 0:
        return ("chain", None)
    p = blocks[bi - 1][-1]
    if p["kind"] == "dw":
        ph = (p["h"] + 2 * (p["k"] // 2) - p["k"]) // p["stride"] + 1
        pc = p["c"]
    else:
        ph, pc = p["h"], p["c_out"]
    if (ph, pc) == (l["h"], c):
        return ("chain", None)
    return ("stage", f"{net}/pooled_b{bi}_{l['h']}x{c}")  # a pool / non-DW/PW layer in between

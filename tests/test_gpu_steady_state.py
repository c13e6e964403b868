"""Steady-state and executed-plan parity (CUDA path vs the oracle, element by element).

(a) Steady state. The persistent tensor-core kernels launch min(tiles, 148) CTAs and loop over
    tiles; a CTA that runs one tile never wraps its X / A / B rings, never alternates its two TMEM
    accumulators and never reuses resident weights across tiles. Every case below has at least
    3 x 148 tiles, so every CTA runs >= 3 tiles and all of that state machinery turns over under an
    oracle check (tolerance of DESIGN.md reading R10; int8 bit-exact).
(b) Executed plans. The committed measured plans (profiles/) are run at a small batch with the
    plan's own tiles; every entry's output is compared with the oracle applied to that entry's
    actual input (the previous entry's GPU output), so each FCM / LBL kernel of the headline plans
    is checked where it runs, without error accumulating along the stack.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import synth
from tests.cases import Case, as_np, compare, oracle_entry

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMS = 148


def _tiles(n, ho, wo, tile, nsplit=1):
    nb = tile.get("tile_n", 1)
    return math.ceil(n / nb) * math.ceil(ho / tile["tile_h"]) * math.ceil(wo / tile["tile_w"]) * nsplit


# ---------------------------------------------------------------- (a) steady state, >= 3 tiles per CTA
# (fmt, n, h, w, c_in, c_out, s, tile, n_split)
DWPW_STEADY = [
    ("bf16", 56, 32, 32, 96, 40, 1, dict(tile_h=8, tile_w=16), 1),            # 128-px tiles, 2 C_in chunks
    ("f16", 56, 32, 32, 96, 40, 1, dict(tile_h=8, tile_w=16), 1),
    ("bf16", 28, 64, 64, 80, 24, 1, dict(tile_h=16, tile_w=16), 1),           # 256-px tiles (2 MMA row blocks)
    ("f16", 28, 64, 64, 80, 24, 1, dict(tile_h=16, tile_w=16), 1),
    ("bf16", 25, 48, 48, 80, 40, 2, dict(tile_h=4, tile_w=8), 1),             # stride 2, ragged last chunk
    ("bf16", 16, 28, 28, 64, 96, 1, dict(tile_h=4, tile_w=8, n_split=2), 2),  # two C_out splits
    ("bf16", 900, 7, 7, 160, 64, 1, dict(tile_h=7, tile_w=7, tile_n=2), 1),   # two images per tile
    ("s8", 56, 32, 32, 160, 48, 1, dict(tile_h=8, tile_w=16), 1),             # int8 (bit-exact)
    ("s8", 25, 48, 48, 96, 32, 2, dict(tile_h=4, tile_w=8), 1),
]


@pytest.mark.parametrize("fmt,n,h,w,ci,co,s,tile,ns", DWPW_STEADY)
def test_dwpw_steady_state(fmt, n, h, w, ci, co, s, tile, ns):
    ho, wo = (h - 1) // s + 1, (w - 1) // s + 1
    assert _tiles(n, ho, wo, tile, ns) >= 3 * SMS
    Case("dwpw", fmt, n, h, w, ci, co, k=3, s=s, tile=tile).check()


@pytest.mark.parametrize("fmt", ["bf16", "f16", "s8"])
@pytest.mark.parametrize("s", [1, 2])
def test_pwdw_r_steady_state(fmt, s):
    # 4x4 output tiles x C_mid slices of 128 bytes: >= 444 (tile, slice) units
    c_in, c_mid = (32, 256) if fmt == "s8" else (24, 128)
    ho = 16
    h = ho * s
    tile = dict(tile_h=4, tile_w=4)
    slices = c_mid // (128 if fmt == "s8" else 64)
    n = math.ceil(3 * SMS / (_tiles(1, ho, ho, tile) * slices))
    assert _tiles(n, ho, ho, tile, slices) >= 3 * SMS
    Case("pwdw", fmt, n, h, h, c_in, c_mid, k=3, s=s, tile=tile).check()


def test_dwpw_f32_3xtf32_steady_state():
    # fp32 DWPW on the tensor-core kernel (T_hi / T_lo commBuffer, resident W / W_lo): >= 3 tiles
    # per CTA, MobileNetV2 block-2 shape with its shortcut
    Case("dwpw", "f32", 8, 56, 56, 144, 24, residual=True).check()


def test_pw_f32_3xtf32_steady_state():
    # fp32 PW on the tensor cores (3xTF32): >= 3 tiles per CTA, 3 C_in chunks, 2 C_out slices
    Case("pw", "f32", 4, 56, 56, 80, 192).check()


@pytest.mark.parametrize("fmt", ["bf16", "f16"])
def test_pwdw_r_wide_halo_steady_state(fmt):
    # 7 x 14 stride-2 output tiles (435 halo rows = 4 MMA row blocks), 32-byte X rows (C_in = 16)
    tile = dict(tile_h=7, tile_w=14)
    ho, wo = 28, 28
    n = math.ceil(3 * SMS / (_tiles(1, ho, wo, tile) * 2))
    assert _tiles(n, ho, wo, tile, 2) >= 3 * SMS
    Case("pwdw", fmt, n, 2 * ho, 2 * wo, 16, 96, k=3, s=2, tile=tile).check()


@pytest.mark.parametrize("fmt", ["bf16", "f16", "s8"])
@pytest.mark.parametrize("c_in,c_out", [(64, 96), (144, 24), (96, 576)])
def test_pw_steady_state(fmt, c_in, c_out):
    # >= 444 row blocks of 128 pixels (M = 16 x 60 x 60 = 57 600)
    assert 16 * 60 * 60 // 128 >= 3 * SMS
    Case("pw", fmt, 16, 60, 60, c_in, c_out).check()


@pytest.mark.parametrize("fmt", ["bf16", "s8"])
@pytest.mark.parametrize("c_in,c_mid,c_out", [(144, 32, 144), (64, 64, 384)])
def test_pwpw_steady_state(fmt, c_in, c_mid, c_out):
    assert 16 * 60 * 60 // 128 >= 3 * SMS
    Case("pwpw", fmt, 16, 60, 60, c_in, c_out, c_mid=c_mid, act_dw=synth.ACT_RELU6).check()


# ---------------------------------------------------------------- (b) the executed (measured) plans
PLANS = [
    ("mobilenet_v2", "bf16", "profiles/r01_plan_mv2_measured.json"),
    ("mobilenet_v1", "s8", "profiles/r01_configs/plan_mobilenet_v1_s8_64.json"),
    ("efficientnet_b0", "s8", "profiles/r01_configs/plan_efficientnet_b0_s8_256.json"),
    ("cvt13", "bf16", "profiles/r01_configs/plan_cvt13_bf16_512.json"),
]


@pytest.mark.parametrize("net,fmt,path", PLANS)
def test_executed_plan_entries_match_oracle(net, fmt, path):
    from oracle import network as onet
    from paper_2404_19331_b200.network import Network
    plan = json.load(open(os.path.join(ROOT, path)))
    assert plan["dtype"] == fmt
    batch = 3
    nw = Network(net, fmt, batch, {"entries": plan["entries"]})
    nw.run()
    torch.cuda.synchronize()
    prm = onet.params(net, fmt)
    kinds = set()
    for e, x_dev, y_dev, r_dev in zip(nw.entries, nw.inputs, nw.outputs, nw.residuals):
        x, y = as_np(x_dev, fmt), as_np(y_dev, fmt)
        ref, mag = oracle_entry(e, nw.layers, prm, x, fmt, None if r_dev is None else as_np(r_dev, fmt))
        compare(y, ref, mag, fmt, f"{net}/{fmt} entry {e['op']} {e['layers']} tile {e.get('tile')}")
        kinds.add(e["op"])
    assert len(kinds) >= 2
    if fmt == "s8":
        # int8: the whole stack is the oracle's stack, bit for bit
        want = onet.forward(net, fmt, 0, batch)
        np.testing.assert_array_equal(as_np(nw.out, fmt), want)

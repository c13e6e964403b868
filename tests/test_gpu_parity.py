"""CUDA path vs the oracle, element by element, on seeded inputs (through the C ABI).

Sizes span several tiles, ragged spatial/channel tails, both strides, k=3/5, every dtype.
"""
import numpy as np
import pytest

import synth
import torch

from oracle import conv as oc
from tests.cases import Case, as_np, compare, stored

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------- configs[0]: the single DWPW layer
@pytest.mark.parametrize("fmt", ["f32", "s8", "bf16", "f16"])
def test_config0_single_dwpw(fmt):
    Case("dwpw", fmt, 1, 14, 14, 16, 32, k=3, s=1).check()


@pytest.mark.parametrize("fmt", ["f32", "s8", "bf16"])
def test_config0_unfused_layers(fmt):
    Case("dw", fmt, 1, 14, 14, 16, k=3, s=1).check()
    Case("pw", fmt, 1, 14, 14, 16, 32).check()


# ---------------------------------------------------------------- DW
@pytest.mark.parametrize("fmt", ["f32", "bf16", "f16", "s8"])
@pytest.mark.parametrize("k,s", [(3, 1), (3, 2), (5, 1), (5, 2), (7, 1), (7, 2)])
def test_dw(fmt, k, s):
    c = 160 if fmt == "s8" else 80
    Case("dw", fmt, 2, 23, 29, c, k=k, s=s).check()


# int8 stride-1 3x3 / 5x5 DW on maps >= 14 x 14 runs on the tensor cores (diagonal weight blocks,
# row-shifted swizzled views of the X tile; tc.cu dw_tc_i8_kernel): partial 128-channel chunks and
# 32-channel groups, 32 / 64 / 128-byte X rows, ragged 16 x 8 tiles, asymmetric pads; bit-exact vs
# the oracle. (Smaller maps and 5x5 with C > 512 take the CUDA-core kernel: last two cases.)
@pytest.mark.parametrize("k", [3, 5])
@pytest.mark.parametrize("n,h,w,c,pads", [
    (1, 17, 19, 16, None),           # one 16-channel group (32-byte rows), ragged tile in both directions
    (2, 23, 29, 144, None),          # 128 + 16 channels (partial chunk)
    (1, 15, 15, 48, (0, 2, 1, 0)),   # asymmetric pads, 64-byte rows, partial 32-channel group
    (3, 14, 14, 256, None),          # MobileNetV2-like map, two chunks
    (1, 30, 14, 96, None),           # 64 + 32 channels in one 128-byte chunk
    (1, 1, 3, 32, None),             # tiny map (CUDA-core kernel)
    (1, 14, 14, 528, None),          # 5x5 with C > 512 on the CUDA-core kernel, 3x3 on the tensor cores
])
def test_dw_int8_tensor_core(k, n, h, w, c, pads):
    Case("dw", "s8", n, h, w, c, k=k, s=1, pads=pads).check()


def test_dw_int8_tensor_core_steady_state():
    # >= 3 tiles per CTA at 2 CTAs per SM: 148 * 2 * 3 spatial tiles of 16 x 8 per 128-channel chunk
    Case("dw", "s8", 24, 56, 56, 128, k=3, s=1).check()


def test_dw_asymmetric_pads_and_tiny():
    Case("dw", "bf16", 1, 1, 1, 16, k=3, s=1).check()
    Case("dw", "bf16", 2, 12, 12, 24, k=3, s=2, pads=(0, 0, 1, 1)).check()
    Case("dw", "s8", 1, 9, 7, 32, k=5, s=1, pads=(1, 2, 3, 0)).check()


def test_dw_nchw():
    import paper_2404_19331_b200 as fcm
    c = Case("dw", "bf16", 2, 11, 13, 24, k=3, s=2)
    ref, mag = c.oracle()
    from tests.cases import device_epi
    x = c.x.permute(0, 3, 1, 2).contiguous().cuda()
    y = fcm.dw(x, stored(c.pd["w"], "bf16").cuda(), 2, None, device_epi(c.pd, "bf16", "cuda"), layout="nchw")
    compare(as_np(y.permute(0, 2, 3, 1), "bf16"), ref, mag, "bf16", "dw nchw")


# ---------------------------------------------------------------- PW
@pytest.mark.parametrize("fmt", ["f32", "bf16", "f16", "s8"])
@pytest.mark.parametrize("c_in,c_out", [(16, 32), (40, 24), (144, 24), (320, 1280), (96, 576)])
def test_pw(fmt, c_in, c_out):
    Case("pw", fmt, 2, 13, 11, c_in, c_out).check()


# ---------------------------------------------------------------- FCM DWPW
@pytest.mark.parametrize("fmt", ["bf16", "f16", "s8", "f32"])
@pytest.mark.parametrize("k,s", [(3, 1), (3, 2), (5, 1), (5, 2)])
def test_dwpw(fmt, k, s):
    c_in, c_out = (160, 48) if fmt == "s8" else (96, 40)
    Case("dwpw", fmt, 3, 23, 21, c_in, c_out, k=k, s=s).check()


@pytest.mark.parametrize("shape", [(4, 7, 7, 160, 320), (2, 14, 14, 576, 96), (1, 28, 28, 32, 16),
                                   (2, 56, 56, 144, 24)])
def test_dwpw_network_shapes_bf16(shape):
    n, h, w, ci, co = shape
    Case("dwpw", "bf16", n, h, w, ci, co, k=3, s=1).check()


@pytest.mark.parametrize("fmt", ["bf16", "f16"])
@pytest.mark.parametrize("act", [synth.ACT_NONE, synth.ACT_RELU, synth.ACT_RELU6])
def test_dwpw_pair_core_acts_and_partial_chunks(fmt, act):
    # column-pair FFMA2 DW core: every activation; C_in = 24 (12 words: 16-lane slots) and
    # 208 = 3 full 64-channel chunks + 16 (8-lane slots); stride 1 and 2
    Case("dwpw", fmt, 2, 17, 19, 24, 40, k=3, s=1, act_dw=act).check()
    Case("dwpw", fmt, 2, 17, 19, 208, 24, k=3, s=2, act_dw=act).check()


@pytest.mark.parametrize("s", [1, 2])
def test_dwpw_odd_and_ragged_tiles(s):
    # odd tile widths leave a single-column last pair; ragged tiles clip at the map edge
    for tile in [dict(tile_h=7, tile_w=7), dict(tile_h=5, tile_w=9), dict(tile_h=13, tile_w=3),
                 dict(tile_h=16 // s, tile_w=8), dict(tile_h=4, tile_w=5, tile_n=3)]:
        Case("dwpw", "bf16", 3, 19, 17, 96, 40, k=3, s=s, tile=tile).check()


def test_dwpw_two_row_block_tiles():
    # pair-core tiles of 129..256 pixels: two M=128 MMA row blocks, direct register epilogue
    # (stride 2 halos of such tiles do not fit two smem stages; the tile chooser never picks them)
    for tile in [dict(tile_h=16, tile_w=16), dict(tile_h=14, tile_w=14), dict(tile_h=28, tile_w=7),
                 dict(tile_h=7, tile_w=7, tile_n=5), dict(tile_h=13, tile_w=11)]:
        Case("dwpw", "bf16", 5, 30, 29, 96, 40, k=3, s=1, tile=tile).check()
    Case("dwpw", "f16", 2, 33, 35, 24, 16, k=3, s=1, tile=dict(tile_h=16, tile_w=16)).check()


def test_dwpw_explicit_tiles_and_splits():
    for tile in [dict(tile_h=4, tile_w=8), dict(tile_h=8, tile_w=16, n_split=2), dict(tile_h=7, tile_w=7, tile_n=2)]:
        Case("dwpw", "bf16", 3, 14, 14, 64, 96, tile=tile).check()


# ---------------------------------------------------------------- FCM PWDW_R
@pytest.mark.parametrize("fmt", ["bf16", "f16", "s8", "f32"])
@pytest.mark.parametrize("k,s", [(3, 1), (3, 2), (5, 1), (5, 2)])
def test_pwdw_r(fmt, k, s):
    c_in, c_mid = (32, 144) if fmt == "s8" else (24, 72)
    Case("pwdw", fmt, 2, 19, 17, c_in, c_mid, k=k, s=s).check()


def test_pwdw_r_border_trap_nonzero_bias():
    """PW bias is nonzero -> T must be zero-padded, not eps_pw(PW(0)) (reading R6)."""
    c = Case("pwdw", "bf16", 1, 9, 9, 16, 64, k=3, s=1)
    c.pp["bias"] = np.full_like(c.pp["bias"], 0.75)
    c.check()


def test_pwdw_r_tiling_invariance_bitwise():
    outs = []
    for tile in [None, dict(tile_h=4, tile_w=4), dict(tile_h=7, tile_w=3), dict(tile_h=14, tile_w=14)]:
        c = Case("pwdw", "bf16", 2, 14, 14, 32, 64, k=3, s=1, tile=tile)
        outs.append(c.gpu())
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


# halo tiles of up to 512 MMA rows (4 row blocks; bf16 / f16) and X boxes staged at the pixel's own
# width (C_in * 2 bytes rounded to 32 / 64, else 128-byte chunks), 4-column DW items incl. tiles
# narrower than 4 columns and ragged maps
@pytest.mark.parametrize("fmt", ["bf16", "f16"])
@pytest.mark.parametrize("c_in,s,h,w,tile", [
    (16, 2, 37, 45, dict(tile_h=7, tile_w=14)),    # R = 15 x 29 = 435, 32-byte X rows
    (24, 2, 33, 30, dict(tile_h=8, tile_w=14)),    # R = 17 x 29 = 493, 64-byte X rows
    (32, 1, 29, 31, dict(tile_h=14, tile_w=28)),   # R = 16 x 30 = 480
    (72, 1, 23, 26, dict(tile_h=16, tile_w=16)),   # R = 324 (3 row blocks), two C_in chunks (64 + 8)
    (16, 1, 13, 11, dict(tile_h=13, tile_w=3)),    # tile narrower than a 4-column DW item
    (40, 2, 21, 9, dict(tile_h=5, tile_w=2)),
])
def test_pwdw_r_wide_halo_narrow_x(fmt, c_in, s, h, w, tile):
    Case("pwdw", fmt, 2, h, w, c_in, 96, k=3, s=s, tile=tile).check()


@pytest.mark.parametrize("fmt", ["bf16", "s8"])
@pytest.mark.parametrize("n_split", [1, 3, 6])
def test_pw_explicit_cout_split(fmt, n_split):
    """The tensor-core PW's C_out split (tile n_split, searched by the measured plan) changes the
    tiling, never the values: oracle parity and bitwise equality with the default split."""
    c = Case("pw", fmt, 2, 13, 11, 48, 384, tile=dict(n_split=n_split))
    c.check()
    d = Case("pw", fmt, 2, 13, 11, 48, 384)
    assert np.array_equal(c.gpu(), d.gpu())


def test_pwdw_r_wide_halo_tiling_invariance_bitwise():
    outs = []
    for tile in [dict(tile_h=4, tile_w=4), dict(tile_h=7, tile_w=14), dict(tile_h=8, tile_w=14), dict(tile_h=15, tile_w=3)]:
        outs.append(Case("pwdw", "bf16", 2, 30, 29, 16, 96, k=3, s=2, tile=tile).gpu())
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


# ---------------------------------------------------------------- GPU self-consistency
def test_int8_fused_equals_unfused_bitwise():
    import paper_2404_19331_b200 as fcm
    from tests.cases import device_epi
    c = Case("dwpw", "s8", 2, 20, 20, 64, 48, k=3, s=2)
    x = c.x.cuda()
    wdw, ed = stored(c.pd["w"], "s8").cuda(), device_epi(c.pd, "s8", "cuda")
    wpk, ep = fcm.pack_pw(stored(c.pp["w"], "s8").cuda()), device_epi(c.pp, "s8", "cuda")
    fused = fcm.dwpw(x, wdw, 2, None, ed, wpk, ep)
    unfused = fcm.pw(fcm.dw(x, wdw, 2, None, ed), wpk, ep)
    assert torch.equal(fused, unfused)


# ---------------------------------------------------------------- error behaviour
def test_abi_errors_on_gpu():
    import paper_2404_19331_b200 as fcm
    from paper_2404_19331_b200._lib import FcmError
    x = torch.zeros(1, 8, 8, 32, dtype=torch.int8, device="cuda")
    w = torch.zeros(3, 3, 32, dtype=torch.int8, device="cuda")
    ep = fcm.Epilogue(mult_q=torch.ones(32, dtype=torch.int32, device="cuda"),
                      shift_q=torch.ones(32, dtype=torch.int32, device="cuda"), zp_in=3)
    with pytest.raises(FcmError) as e:
        fcm.dw(x, w, 1, None, ep)
    assert e.value.status == -3  # nonzero input zero point: FCM_E_UNSUPPORTED on the GPU path


# ---------------------------------------------------------------- unaligned channel pitch (CUDA-core paths)
# EfficientNet-B0 int8 has C = 24 / 40: a 24- or 40-byte NHWC pitch, which TMA cannot address.
@pytest.mark.parametrize("fmt", ["s8", "bf16"])
def test_unaligned_pitch_layers(fmt):
    Case("dw", fmt, 2, 13, 11, 40 if fmt == "s8" else 12, k=5, s=2).check()
    Case("pw", fmt, 2, 9, 7, 144, 40 if fmt == "s8" else 12).check()
    Case("dwpw", fmt, 2, 14, 14, 240 if fmt == "s8" else 36, 40 if fmt == "s8" else 12, k=5, s=1).check()
    Case("pwdw", fmt, 2, 15, 13, 24 if fmt == "s8" else 12, 144 if fmt == "s8" else 36, k=5, s=2).check()


# ---------------------------------------------------------------- round-1 kernel variants
@pytest.mark.parametrize("fmt", ["bf16", "f16", "s8"])
@pytest.mark.parametrize("c_out", [16, 96, 144, 192, 320])
def test_pw_epilogue_groups(fmt, c_out):
    # 128-byte column chunks per tile: 1 (4 epilogue groups), 2 (2 groups x 2 accumulators),
    # 3 (2 groups x 1 accumulator, 2 + 1 chunks), >= 4 (1 group); M spans several 128-row tiles
    Case("pw", fmt, 3, 17, 13, 64 if fmt != "s8" else 128, c_out).check()


@pytest.mark.parametrize("fmt,c", [("s8", 32), ("s8", 16), ("bf16", 24), ("bf16", 16), ("f32", 8), ("f16", 40)])
@pytest.mark.parametrize("s", [1, 2])
def test_dw_lane_groups_partial_channel_groups(fmt, c, s):
    # a 128-byte channel group with 8 or 16 valid words: 2-4 output columns per warp
    Case("dw", fmt, 2, 21, 19, c, k=3, s=s).check()


@pytest.mark.parametrize("fmt,c_in,c_out", [("s8", 24, 40), ("s8", 40, 24), ("s8", 24, 36), ("bf16", 12, 36),
                                            ("f32", 7, 9), ("f32", 16, 12), ("bf16", 6, 10)])
def test_pw_simt_vector_and_scalar_paths(fmt, c_in, c_out):
    # pitches TMA cannot address: 8-byte staging + vector stores (int8 via __dp4a) when the row
    # pitch is a multiple of 8 bytes and C_out of 4, element-wise otherwise
    Case("pw", fmt, 2, 15, 13, c_in, c_out).check()


@pytest.mark.parametrize("fmt", ["s8", "f16"])
def test_dwpw_lane_groups_non_pair_path(fmt):
    # int8 3x3 / fp16 5x5 DWPW with partly filled C_in chunks (lane groups in the non-pair DW warps)
    k = 3 if fmt == "s8" else 5
    Case("dwpw", fmt, 2, 17, 15, 160 if fmt == "s8" else 72, 48, k=k, s=1).check()
    Case("dwpw", fmt, 2, 17, 15, 32, 48, k=k, s=2).check()


# ---------------------------------------------------------------- FCM PWPW
@pytest.mark.parametrize("fmt", ["bf16", "f16", "s8"])
@pytest.mark.parametrize("c_in,c_mid,c_out", [(144, 24, 144), (64, 64, 384), (96, 96, 576), (32, 128, 200),
                                              (576, 96, 24)])
def test_pwpw(fmt, c_in, c_mid, c_out):
    # M spans several 128-row tiles plus a ragged tail; C_out in several GEMM2 slices
    if fmt == "s8" and (c_in % 16 or c_mid % 16 or c_out % 16):
        pytest.skip("int8 tensor-core path needs 16-byte pitches")
    Case("pwpw", fmt, 3, 13, 11, c_in, c_out, c_mid=c_mid, act_dw=synth.ACT_RELU6).check()


def test_pwpw_unsupported_cases_fail_loudly():
    import paper_2404_19331_b200 as fcm
    from paper_2404_19331_b200._lib import FcmError
    with pytest.raises(FcmError, match="UNSUPPORTED"):
        Case("pwpw", "f32", 1, 4, 4, 16, 16, c_mid=16).check()
    with pytest.raises(FcmError, match="UNSUPPORTED"):
        Case("pwpw", "bf16", 1, 4, 4, 16, 16, c_mid=160).check()


@pytest.mark.parametrize("act,zp_out,qmin,shift_drop", [(0, 0, -128, 0), (2, 0, 0, 10), (0, 7, -100, 0),
                                                        (1, 0, 0, 12), (0, -3, -128, 9), (0, 0, -128, 7)])
@pytest.mark.parametrize("s,tile", [(1, None), (1, {"tile_h": 5, "tile_w": 7}), (2, {"tile_h": 3, "tile_w": 9})])
def test_dw_int8_pair_core_requant_and_clamp_paths(act, zp_out, qmin, shift_drop, s, tile):
    """The int8 FFMA2 DW core (dw3_pair_i8): saturating-pack clamps (qmin -128 / 0), the generic
    clamp (other qmin, nonzero zp_out), the 64-bit requantiser (shifts <= 32, obtained by dropping
    the shift and the multiplier by the same power of two), and odd tile widths whose last column
    pair is half dead. Bit-exact against the oracle."""
    import numpy as np
    c = Case("dw", "s8", 2, 19, 23, 96, k=3, s=s, tile=tile, act_dw=act)
    p = c.pd
    p["zp_out"], p["qmin"] = zp_out, qmin
    if shift_drop:
        sh = np.asarray(p["shift_q"], dtype=np.int64)
        m = np.asarray(p["mult_q"], dtype=np.int64)
        p["shift_q"] = sh - shift_drop
        p["mult_q"] = m >> shift_drop
        assert (p["shift_q"] <= 32).any()
    c.check()


@pytest.mark.parametrize("fmt,c", [("s8", 728), ("s8", 40), ("s8", 12), ("bf16", 36), ("bf16", 6), ("f32", 5),
                                   ("f16", 30)])
@pytest.mark.parametrize("k,s", [(3, 1), (3, 2), (5, 1), (7, 2)])
def test_dw_cp_async_staging_unaligned_pitch(fmt, c, k, s):
    """Pixel pitches that are multiples of 4 (8) bytes but not 16 (Xception int8 C = 728): the
    tiled DW kernel stages the halo with cp.async instead of TMA, zero-filling outside the image
    and past C; the cores are unchanged (int8 bit-exact, floats within tolerance)."""
    Case("dw", fmt, 2, 11, 13, c, k=k, s=s).check()
    Case("dw", fmt, 1, 9, 10, c, k=k, s=s, tile={"tile_h": 3, "tile_w": 5}).check()


@pytest.mark.parametrize("op", ["dw", "dwpw"])
@pytest.mark.parametrize("s", [1, 2])
@pytest.mark.parametrize("shift", [47, 48])
def test_int8_dw_large_bias_q(op, s, shift):
    """int8 DW with |bias_q| in [1, 2) x 2^22 .. 2^23 (any int32 is legal, fcm.h): the FFMA2 DW
    cores accumulate the taps exactly in fp32 (|sum| < 2^18) and add bias_q in int32 afterwards.
    Shifts 47 / 48 (scale ~2^-17 / 2^-18) keep the outputs unsaturated with zp_out = 0, so a bias
    folded into the fp32 accumulator (exact int conversion only below 2^22) would show. Bit-exact."""
    import numpy as np
    c = Case(op, "s8", 2, 19, 23, 96, 48, k=3, s=s, act_dw=synth.ACT_NONE) if op == "dwpw" else \
        Case(op, "s8", 2, 19, 23, 96, k=3, s=s, act_dw=synth.ACT_NONE)
    p = c.pd
    rng = np.random.default_rng(shift)
    nc = len(p["bias_q"])
    mag = rng.integers(1 << 22, 1 << (shift - 24), size=nc)
    p["bias_q"] = (mag * rng.choice([-1, 1], size=nc)).astype(np.int64)
    p["shift_q"] = np.full(nc, shift, dtype=np.int64)
    p["zp_out"], p["qmin"], p["qmax"] = 0, -128, 127
    t = oc.dw(as_np(c.x, "s8"), p["w"], s, c.pads, p, "s8")
    assert (np.abs(t) < 127).mean() > 0.9 and (np.abs(t) > 8).mean() > 0.5  # unsaturated, bias-driven
    c.check()

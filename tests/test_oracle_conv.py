"""Pins for oracle/conv.py: hand vectors, an independent pure-Python brute force, torch CPU
float64 conv2d (textbook routine), the depthwise-separable factorisation identity
and the PWDW border semantics (reading R6)."""
import itertools
import json
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import conv
from oracle.numerics import requant

GOLD = os.path.join(os.path.dirname(__file__), "golden")
rng = np.random.default_rng(11)


def brute_grouped_conv(x, wt, groups, stride, pads):
    """Generic direct grouped convolution, pure Python (tiny inputs only).
    x: nested [N][H][W][Cin]; wt[i][j][ci_in_group][co]; correlation semantics."""
    n_, h, w, cin = len(x), len(x[0]), len(x[0][0]), len(x[0][0][0])
    k = len(wt)
    cout = len(wt[0][0][0])
    pt, pl, pb, pr = pads
    ho, wo = (h + pt + pb - k) // stride + 1, (w + pl + pr - k) // stride + 1
    gin, gout = cin // groups, cout // groups
    out = [[[[0 for _ in range(cout)] for _ in range(wo)] for _ in range(ho)] for _ in range(n_)]
    for n, y, xx, co in itertools.product(range(n_), range(ho), range(wo), range(cout)):
        g = co // gout
        s = 0
        for i, j, c in itertools.product(range(k), range(k), range(gin)):
            yy, xi = y * stride - pt + i, xx * stride - pl + j
            if 0 <= yy < h and 0 <= xi < w:
                s += x[n][yy][xi][g * gin + c] * wt[i][j][c][co]
        out[n][y][xx][co] = s
    return np.array(out)


def test_all_ones_dw():
    g = json.load(open(os.path.join(GOLD, "worked_vectors.json")))["all_ones_dw"]
    x = np.ones((1, 3, 3, 1))
    out = conv.dw_acc(x, np.ones((3, 3, 1)), 1, (1, 1, 1, 1))
    assert out[0, :, :, 0].tolist() == g["expect"]


def test_impulse_gives_flipped_kernel():
    x = np.zeros((1, 7, 7, 1))
    x[0, 3, 3, 0] = 1.0
    w = np.arange(1, 10, dtype=np.float64).reshape(3, 3, 1)
    out = conv.dw_acc(x, w, 1, (1, 1, 1, 1))[0, :, :, 0]
    assert np.array_equal(out[2:5, 2:5], w[::-1, ::-1, 0])  # correlation => flipped kernel
    assert out.sum() == w.sum()


def test_identities():
    x = rng.uniform(-1, 1, (2, 5, 6, 3))
    wc = np.zeros((3, 3, 3))
    wc[1, 1, :] = 1
    assert np.array_equal(conv.dw_acc(x, wc, 1, (1, 1, 1, 1)), x)
    assert np.array_equal(conv.pw_acc(x, np.eye(3)), x)


def test_stride2_hand_table():
    x = np.arange(16, dtype=np.float64).reshape(1, 4, 4, 1)
    out = conv.dw_acc(x, np.ones((3, 3, 1)), 2, (1, 1, 1, 1))[0, :, :, 0]
    # outputs at input centres (0,0),(0,2),(2,0),(2,2): sums of the clipped 3x3 windows
    assert out.tolist() == [[0 + 1 + 4 + 5, 1 + 2 + 3 + 5 + 6 + 7],
                            [4 + 5 + 8 + 9 + 12 + 13, 5 + 6 + 7 + 9 + 10 + 11 + 13 + 14 + 15]]


@pytest.mark.parametrize("k,s,pads", [(3, 1, (1, 1, 1, 1)), (3, 2, (1, 1, 1, 1)), (5, 2, (2, 2, 2, 2)),
                                      (3, 2, (0, 0, 1, 1)), (5, 1, (1, 2, 3, 0)), (7, 1, (3, 3, 3, 3)),
                                      (7, 2, (3, 2, 1, 3))])
def test_dw_brute_force_int(k, s, pads):
    x = rng.integers(-128, 128, (2, 6, 7, 3))
    w = rng.integers(-127, 128, (k, k, 3))
    wt = [[[[int(w[i, j, c]) if c == co else 0 for co in range(1)] for c in range(1)] for j in range(k)]
          for i in range(k)]
    # DW as a grouped conv with groups=C: per-group weight [k][k][1][1] -> assemble [k][k][1][C]
    wt = [[[[int(w[i, j, co]) for co in range(3)]] for j in range(k)] for i in range(k)]
    ref = brute_grouped_conv(x.tolist(), wt, 3, s, pads)
    assert np.array_equal(conv.dw_acc(x.astype(np.int64), w.astype(np.int64), s, pads), ref)


def test_pw_brute_force_int():
    x = rng.integers(-128, 128, (1, 3, 4, 5))
    w = rng.integers(-127, 128, (5, 6))
    wt = [[[[int(w[c, co]) for co in range(6)] for c in range(5)]]]
    assert np.array_equal(conv.pw_acc(x.astype(np.int64), w.astype(np.int64)),
                          brute_grouped_conv(x.tolist(), wt, 1, 1, (0, 0, 0, 0)))


@pytest.mark.parametrize("k,s,p", [(3, 1, 1), (3, 2, 1), (5, 1, 2), (5, 2, 2), (7, 1, 3), (7, 2, 3)])
def test_dw_matches_torch_conv2d_f64(k, s, p):
    x = rng.uniform(-1, 1, (2, 11, 9, 8))
    w = rng.uniform(-1, 1, (k, k, 8))
    ref = F.conv2d(torch.from_numpy(x).permute(0, 3, 1, 2), torch.from_numpy(w).permute(2, 0, 1)[:, None],
                   stride=s, padding=p, groups=8).permute(0, 2, 3, 1).numpy()
    assert np.allclose(conv.dw_acc(x, w, s, (p, p, p, p)), ref, rtol=1e-13, atol=1e-13)


def test_pw_matches_torch_conv2d_f64():
    x = rng.uniform(-1, 1, (2, 5, 7, 12))
    w = rng.uniform(-1, 1, (12, 20))
    ref = F.conv2d(torch.from_numpy(x).permute(0, 3, 1, 2), torch.from_numpy(w.T.copy())[:, :, None, None])
    assert np.allclose(conv.pw_acc(x, w), ref.permute(0, 2, 3, 1).numpy(), rtol=1e-13, atol=1e-13)


def _std_conv(x, wstd, s, p):
    """torch float64 standard conv; wstd[i,j,ci,co]."""
    return F.conv2d(torch.from_numpy(x).permute(0, 3, 1, 2), torch.from_numpy(wstd).permute(3, 2, 0, 1),
                    stride=s, padding=p).permute(0, 2, 3, 1).numpy()


@pytest.mark.parametrize("k,s", [(3, 1), (3, 2), (5, 1)])
def test_dsc_factorisation_identity(k, s):
    """DW followed by PW (a depthwise-separable conv) is a standard conv with the
    factorised weight W[i,j,ci,co] = Wdw[i,j,ci] * Wpw[ci,co] (NONE epilogue, no rounding)."""
    x = rng.uniform(-1, 1, (2, 9, 10, 6))
    wdw, wpw = rng.uniform(-1, 1, (k, k, 6)), rng.uniform(-1, 1, (6, 7))
    p = k // 2
    none = {"act": 0}
    got = conv.dwpw(x, wdw, s, (p,) * 4, none, wpw, none, "f64")
    ref = _std_conv(x, wdw[:, :, :, None] * wpw[None, None], s, p)
    assert np.allclose(got, ref, rtol=1e-12, atol=1e-12)


def test_pwdw_factorisation_and_border_semantics():
    """PW then DW without PW bias = standard conv with W[i,j,ci,co] = Wpw[ci,co]*Wdw[i,j,co].
    With a PW bias the identity breaks at the image border ONLY (DW pads T, not X)."""
    x = rng.uniform(-1, 1, (1, 8, 8, 4))
    wpw, wdw = rng.uniform(-1, 1, (4, 5)), rng.uniform(-1, 1, (3, 3, 5))
    none = {"act": 0}
    got = conv.pwdw(x, wpw, none, wdw, 1, (1,) * 4, none, "f64")
    ref = _std_conv(x, wpw[None, None] * wdw[:, :, None, :], 1, 1)
    assert np.allclose(got, ref, rtol=1e-12, atol=1e-12)
    b = {"act": 0, "bias": rng.uniform(0.5, 1.0, 5)}
    got_b = conv.pwdw(x, wpw, b, wdw, 1, (1,) * 4, none, "f64")
    # interior: bias enters through all 9 taps; border: through fewer taps
    interior_ref = ref[:, 1:-1, 1:-1, :] + (b["bias"][None, :] * wdw.reshape(9, 5)).sum(0)
    assert np.allclose(got_b[:, 1:-1, 1:-1, :], interior_ref, rtol=1e-12, atol=1e-12)
    corner_ref = ref[0, 0, 0, :] + (b["bias"] * wdw[1:, 1:, :].reshape(4, 5)).sum(0)
    assert np.allclose(got_b[0, 0, 0, :], corner_ref, rtol=1e-12, atol=1e-12)


def test_pwdw_border_vector():
    g = json.load(open(os.path.join(GOLD, "worked_vectors.json")))["pwdw_border"]
    x = np.zeros((1, 3, 3, 1))
    out = conv.pwdw(x, np.ones((1, 1)), {"act": 0, "bias": np.ones(1)}, np.ones((3, 3, 1)), 1, (1,) * 4,
                    {"act": 0}, "f64")
    assert out[0, :, :, 0].tolist() == g["expect_pad_T"]
    assert out[0, :, :, 0].tolist() != g["wrong_pad_X"]


def test_int8_dwpw_worked_vector():
    g = json.load(open(os.path.join(GOLD, "worked_vectors.json")))["int8_dwpw"]
    x = np.array(g["x"])[None]
    pdw = dict(bias_q=np.array(g["dw_bias_q"]), mult_q=g["dw_mult"], shift_q=g["dw_shift"], zp_in=0, zp_out=0,
               qmin=g["dw_qmin"], qmax=g["dw_qmax"])
    ppw = dict(bias_q=np.array(g["pw_bias_q"]), mult_q=g["pw_mult"], shift_q=g["pw_shift"], zp_in=0, zp_out=0,
               qmin=g["pw_qmin"], qmax=g["pw_qmax"])
    wdw, wpw = np.array(g["w_dw"]), np.array(g["w_pw"])
    acc = conv.dw_acc(x, wdw, 1, (1,) * 4) + pdw["bias_q"]
    assert acc[0].tolist() == g["dw_acc_plus_bias"]
    t = conv.dw(x, wdw, 1, (1,) * 4, pdw, "s8")
    assert t[0].tolist() == g["t"]
    y = conv.dwpw(x, wdw, 1, (1,) * 4, pdw, wpw, ppw, "s8")
    assert y[0].tolist() == g["y"]
    # independent brute force of the same chain with Python ints
    wt = [[[[int(wdw[i, j, co]) for co in range(2)]] for j in range(3)] for i in range(3)]
    acc_b = brute_grouped_conv(x.tolist(), wt, 2, 1, (1,) * 4) + pdw["bias_q"]
    t_b = np.clip([[[(2 * int(a) * g["dw_mult"] + (1 << g["dw_shift"])) >> (g["dw_shift"] + 1) for a in row]
                    for row in plane] for plane in acc_b[0]], 0, 127)
    assert t_b.tolist() == g["t"]


def test_int8_zero_point_padding():
    """int8 with zp_in != 0: an out-of-image tap holds the zero point, i.e. contributes 0."""
    x = rng.integers(-128, 128, (1, 5, 5, 2))
    w = rng.integers(-127, 128, (3, 3, 2))
    zp = 7
    p = dict(bias_q=np.zeros(2, np.int64), mult_q=1 << 30, shift_q=30, zp_in=zp, zp_out=0, qmin=-10 ** 9,
             qmax=10 ** 9)
    got = conv.dw(x, w, 1, (1,) * 4, p, "s8")  # mult/shift = 1.0 exactly
    xz = np.full((1, 7, 7, 2), zp)
    xz[:, 1:6, 1:6] = x
    ref = conv.dw_acc(xz - zp, w, 1, (0,) * 4)
    assert np.array_equal(got, ref)


def test_linearity_float():
    x1, x2 = rng.uniform(-1, 1, (2, 2, 6, 6, 4))
    w = rng.uniform(-1, 1, (3, 3, 4))
    a = conv.dw_acc(2.0 * x1 - 3.0 * x2, w, 2, (1,) * 4)
    b = 2.0 * conv.dw_acc(x1, w, 2, (1,) * 4) - 3.0 * conv.dw_acc(x2, w, 2, (1,) * 4)
    assert np.allclose(a, b, rtol=1e-12, atol=1e-12)


def test_epilogue_float_rounding_and_act():
    acc = np.array([[[[7.0, -1.0, 3.0]]]])
    p = {"scale": np.array([1.0, 2.0, 0.5]), "bias": np.array([0.0, 0.5, 0.25]), "act": 2}
    out = conv.epilogue_float(acc, p, "f32")
    assert out.ravel().tolist() == [6.0, 0.0, 1.75]  # RELU6 clamps 7->6, -1.5->0
    p1 = {"act": 1}
    assert conv.epilogue_float(np.array([1 + 2 ** -9, -2.0]), p1, "bf16").tolist() == [1.0, 0.0]


def test_pwpw_factorisation_identity():
    # PWPW with identity epilogues and no rounding is one 1x1 conv with W1 . W2: checked
    # against torch's fp64 conv2d with the product weight (a different route than pw(pw(.)))
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, (2, 5, 4, 6))
    w1, w2 = rng.uniform(-1, 1, (6, 9)), rng.uniform(-1, 1, (9, 7))
    ident = dict(act=0, scale=None, bias=None)
    got = conv.pwpw(x, w1, ident, w2, ident, "f64")
    wf = torch.from_numpy(w1 @ w2).t()[:, :, None, None]
    want = F.conv2d(torch.from_numpy(x).permute(0, 3, 1, 2), wf).permute(0, 2, 3, 1).numpy()
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)
    # with a bias and RELU between the two PWs the product form no longer holds -> T is materialised
    p1 = dict(act=1, scale=None, bias=np.full(9, -0.5))
    assert not np.allclose(conv.pwpw(x, w1, p1, w2, ident, "f64"), want)


def test_pwpw_int8_intermediate_is_requantised():
    # the int8 commBuffer is requantised before the second PW: brute force with Python ints
    rng = np.random.default_rng(11)
    x = rng.integers(-128, 128, (1, 2, 3, 4))
    w1, w2 = rng.integers(-127, 128, (4, 3)), rng.integers(-127, 128, (3, 5))
    p1 = dict(act=2, bias_q=np.array([5, -7, 0]), mult_q=np.array([1 << 30] * 3), shift_q=np.array([36] * 3),
              zp_in=0, zp_out=0, qmin=0, qmax=96)
    p2 = dict(act=0, bias_q=np.zeros(5, np.int64), mult_q=np.array([1 << 30] * 5), shift_q=np.array([33] * 5),
              zp_in=0, zp_out=0, qmin=-128, qmax=127)
    got = conv.pwpw(x, w1, p1, w2, p2, "s8")
    for n, yy, xx in itertools.product(range(1), range(2), range(3)):
        t = []
        for c in range(3):
            acc = sum(int(x[n, yy, xx, i]) * int(w1[i, c]) for i in range(4)) + int(p1["bias_q"][c])
            r = (acc * (1 << 30) + (1 << 35)) >> 36
            t.append(min(max(r, 0), 96))
        for o in range(5):
            acc = sum(t[c] * int(w2[c, o]) for c in range(3))
            r = (acc * (1 << 30) + (1 << 32)) >> 33
            assert got[n, yy, xx, o] == min(max(r, -128), 127)


# ---------------------------------------------------------------- SURVEY §8(f) rank 4 epilogues
def test_silu_gelu_match_torch_and_closed_forms():
    """SiLU / GELU of the oracle epilogue vs torch's own F.silu / F.gelu (exact erf form) in fp64,
    plus closed-form special values and GELU's odd-part identity gelu(v) - gelu(-v) = v."""
    v = np.concatenate([np.linspace(-12, 12, 2401), [-800.0, -40.0, 0.0, 40.0, 800.0]])
    tv = torch.from_numpy(v)
    silu = conv.act_float(v, conv.ACT_SILU)
    gelu = conv.act_float(v, conv.ACT_GELU)
    np.testing.assert_allclose(silu, F.silu(tv).numpy(), rtol=1e-15, atol=1e-300)
    np.testing.assert_allclose(gelu, F.gelu(tv).numpy(), rtol=1e-12, atol=1e-15)  # erf tails differ by ulps
    assert conv.act_float(np.array([0.0]), conv.ACT_SILU)[0] == 0.0
    assert conv.act_float(np.array([0.0]), conv.ACT_GELU)[0] == 0.0
    assert conv.act_float(np.array([40.0]), conv.ACT_SILU)[0] == 40.0 / (1.0 + np.exp(-40.0))
    assert abs(conv.act_float(np.array([1.0]), conv.ACT_SILU)[0] - 1.0 / (1.0 + np.e ** -1.0)) < 1e-16
    # sigmoid(0) = 1/2 => silu'(0) = 1/2 ; Phi(1) = 0.8413447460685429 (normal table)
    assert abs(conv.act_float(np.array([1.0]), conv.ACT_GELU)[0] - 0.8413447460685429) < 1e-15
    np.testing.assert_allclose(conv.act_float(v, conv.ACT_GELU) - conv.act_float(-v, conv.ACT_GELU), v, atol=1e-12)
    assert conv.act_float(np.array([-800.0]), conv.ACT_SILU)[0] == 0.0  # -800 * e^-800 underflows


def test_residual_add_is_after_activation():
    """y = round(act(acc*s + b) + r): with act = RELU6 and fp64 the result is exactly the
    activation output plus r (the shortcut is not clipped), and a zero residual changes nothing."""
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, (2, 5, 4, 8))
    w = rng.uniform(-1, 1, (8, 6))
    r = rng.uniform(-10, 10, (2, 5, 4, 6))
    p = {"act": conv.ACT_RELU6, "scale": rng.uniform(0.5, 4, 6), "bias": rng.uniform(-2, 2, 6)}
    base = conv.pw(x, w, p, "f64")
    withr = conv.pw(x, w, dict(p, residual=r), "f64")
    np.testing.assert_array_equal(withr, base + r)
    assert withr.max() > 6.0 or withr.min() < 0.0  # the sum is outside the RELU6 range: not clipped
    np.testing.assert_array_equal(conv.pw(x, w, dict(p, residual=np.zeros_like(r)), "f64"), base)
    # bf16 rounding happens once, after the add
    bf = conv.pw(x, w, dict(p, residual=r), "bf16")
    ref = torch.from_numpy(base + r).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(bf, ref)

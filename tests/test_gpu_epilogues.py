"""GPU parity of the whole-network epilogues: SiLU / GELU activations and the
residual (shortcut) add, element-wise against the oracle through the C ABI.

Shapes cover ragged channel tails (C_out = 24 / 40: half-filled 16-column groups), M not a multiple
of 128, stride 2, and launches with more than 3 x 148 tiles (every persistent CTA loops)."""
import pytest
import torch

import synth
from tests.cases import Case

pytestmark = pytest.mark.gpu

ACTS = [synth.ACT_SILU, synth.ACT_GELU]


@pytest.mark.parametrize("fmt", ["bf16", "f16", "f32"])
@pytest.mark.parametrize("act", ACTS)
def test_dw_act(fmt, act):
    Case("dw", fmt, 2, 15, 13, 72, act_dw=act, s=1).check()
    Case("dw", fmt, 2, 15, 13, 72, act_dw=act, s=2).check()


@pytest.mark.parametrize("fmt", ["bf16", "f16", "f32"])
@pytest.mark.parametrize("act", ACTS)
def test_pw_act(fmt, act):
    Case("pw", fmt, 2, 13, 11, 40, 96, act_pw=act).check()


@pytest.mark.parametrize("fmt", ["bf16", "f16", "f32"])
@pytest.mark.parametrize("act", ACTS)
@pytest.mark.parametrize("s", [1, 2])
def test_dwpw_act(fmt, act, s):
    # act on both convs: the DW stage's (fused, on-chip T) and the PW epilogue's
    Case("dwpw", fmt, 2, 15, 13, 96, 40, s=s, act_dw=act, act_pw=act).check()


@pytest.mark.parametrize("fmt", ["bf16", "f16"])
@pytest.mark.parametrize("act", ACTS)
def test_pwdw_r_act(fmt, act):
    c = Case("pwdw", fmt, 2, 15, 13, 24, 72, act_dw=act)
    c.pp["act"] = act  # the PW producing T, too
    c.check()


@pytest.mark.parametrize("fmt", ["bf16", "f16"])
@pytest.mark.parametrize("act", ACTS)
def test_pwpw_act(fmt, act):
    Case("pwpw", fmt, 2, 14, 14, 192, 96, c_mid=64, act_dw=act, act_pw=act).check()


@pytest.mark.parametrize("fmt", ["bf16", "f16", "f32"])
@pytest.mark.parametrize("c_in,c_out", [(144, 24), (96, 40), (384, 64)])
def test_pw_residual(fmt, c_in, c_out):
    Case("pw", fmt, 3, 17, 15, c_in, c_out, residual=True).check()


@pytest.mark.parametrize("fmt", ["bf16", "f16", "f32"])
@pytest.mark.parametrize("shape", [(2, 15, 13, 144, 24), (2, 14, 14, 384, 64), (3, 7, 7, 576, 96)])
def test_dwpw_residual(fmt, shape):
    n, h, w, ci, co = shape
    Case("dwpw", fmt, n, h, w, ci, co, residual=True).check()


def test_dwpw_residual_steady_state_bf16():
    # > 3 x 148 tiles per launch: MobileNetV2 block-2 shape (56^2 x 144 -> 24) at batch 8
    Case("dwpw", "bf16", 8, 56, 56, 144, 24, residual=True, tile={"tile_h": 28, "tile_w": 8}).check()


@pytest.mark.parametrize("fmt", ["bf16", "f16"])
def test_pwpw_residual(fmt):
    Case("pwpw", fmt, 3, 14, 14, 64, 64, c_mid=128, residual=True).check()


def test_residual_rejected_where_undefined():
    import paper_2404_19331_b200 as fcm
    from paper_2404_19331_b200._lib import FcmError, FCM_E_UNSUPPORTED
    dev = "cuda:0"
    x = torch.zeros(1, 8, 8, 32, dtype=torch.bfloat16, device=dev)
    r = torch.zeros(1, 8, 8, 32, dtype=torch.bfloat16, device=dev)
    wdw = torch.zeros(3, 3, 32, dtype=torch.bfloat16, device=dev)
    with pytest.raises(FcmError) as e:
        fcm.dw(x, wdw, 1, None, fcm.Epilogue(residual=r))
    assert e.value.status == FCM_E_UNSUPPORTED
    wpk = fcm.pack_pw(torch.zeros(32, 32, dtype=torch.bfloat16, device=dev))
    with pytest.raises(FcmError) as e:
        fcm.pwdw_r(x, wpk, fcm.Epilogue(), wdw, 1, None, fcm.Epilogue(residual=r))
    assert e.value.status == FCM_E_UNSUPPORTED
    xi = torch.zeros(1, 8, 8, 32, dtype=torch.int8, device=dev)
    one = torch.ones(32, dtype=torch.int32, device=dev)
    with pytest.raises(FcmError) as e:
        fcm.pw(xi, fcm.pack_pw(torch.zeros(32, 32, dtype=torch.int8, device=dev)),
               fcm.Epilogue(mult_q=one << 30, shift_q=one * 31, residual=xi))
    assert e.value.status == FCM_E_UNSUPPORTED

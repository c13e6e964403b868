"""Whole DW/PW stacks on the GPU through the C ABI (MobileNetV2 / EfficientNet-B0, synthetic).

* int8: FCMs are bit-exact with the unfused composition (reading R2), so a FusePlanner plan and
  the all-LBL plan of the same stack must give identical bytes.
* Programmatic dependent launch (FCM_PDL) changes only launch overlap, never results: the
  bf16 stack output is bitwise identical with it on and off (separate processes: the switch is
  read once per process).
"""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lbl_plan(plan):
    ents = [dict(e) for e in plan["candidates"]["lbl"]]
    return {"entries": ents, "totals": plan["totals"], "mode": plan["mode"]}


@pytest.mark.parametrize("net,dt,batch", [("efficientnet_b0", "s8", 3), ("mobilenet_v1", "s8", 2)])
def test_int8_stack_fused_plan_equals_layer_by_layer(net, dt, batch):
    import paper_2404_19331_b200 as fcm
    from paper_2404_19331_b200.network import Network, model_json
    plan = fcm.plan(model_json(net, dt, batch))
    assert plan["totals"]["fused_pairs"] > 0
    a = Network(net, dt, batch, plan)
    a.run()
    b = Network(net, dt, batch, _lbl_plan(plan))
    b.run()
    torch.cuda.synchronize()
    assert torch.equal(a.out.cpu(), b.out.cpu())


_SCRIPT = r"""
import sys, torch
sys.path.insert(0, {root!r})
import paper_2404_19331_b200 as fcm
from paper_2404_19331_b200.network import Network, model_json
plan = fcm.plan(model_json("mobilenet_v2", "bf16", 4))
n = Network("mobilenet_v2", "bf16", 4, plan)
g = n.capture()
g.replay(); g.replay()
torch.cuda.synchronize()
torch.save(n.out.cpu(), sys.argv[1])
"""


def test_pdl_does_not_change_results(tmp_path):
    outs = []
    for pdl in ("0", "1"):
        f = tmp_path / f"out{pdl}.pt"
        env = dict(os.environ, FCM_PDL=pdl)
        r = subprocess.run([sys.executable, "-c", _SCRIPT.format(root=ROOT), str(f)], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(torch.load(f))
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("net,dt,batch", [("mobilenet_v2", "bf16", 2), ("mobilenet_v1", "s8", 2)])
def test_stack_with_pwpw_equals_layer_by_layer(net, dt, batch):
    # replace PW -> PW chain pairs of the all-LBL plan by FCM PWPW entries: identical bytes (the
    # PWPW kernel rounds / requantises T exactly like the unfused PW epilogue)
    import paper_2404_19331_b200 as fcm
    from paper_2404_19331_b200.autotune import pwpw_candidates
    from paper_2404_19331_b200.network import Network, model_json
    plan = fcm.plan(model_json(net, dt, batch))
    lbl = _lbl_plan(plan)
    probe = Network(net, dt, batch, {"entries": []})
    cands = {tuple(c["layers"]): c for c in pwpw_candidates(model_json(net, dt, batch), probe, dt, batch)}
    ents, i, used = [], 0, 0
    while i < len(lbl["entries"]):
        e = lbl["entries"][i]
        if i + 1 < len(lbl["entries"]):
            key = (e["layers"][0], lbl["entries"][i + 1]["layers"][0])
            if key in cands and probe.layers[key[0]]["c_out"] <= 128 and probe.layers[key[0]]["c_out"] % 16 == 0:
                ents.append(cands[key])
                i += 2
                used += 1
                continue
        ents.append(e)
        i += 1
    if used == 0:
        pytest.skip("no PW -> PW chain pair in this stack")
    a = Network(net, dt, batch, dict(lbl, entries=ents))
    a.run()
    b = Network(net, dt, batch, lbl)
    b.run()
    torch.cuda.synchronize()
    assert torch.equal(a.out.cpu(), b.out.cpu())


@pytest.mark.parametrize("net", ["xception", "ceit_leff", "cmt_irffn", "proxylessnas_gpu"])
def test_fusion_case_networks_int8_match_oracle(net):
    """the paper's other fusion-case networks (XCe, CeiT, CMT)
    as DW/PW stacks. int8: the planned (fused) stack == the all-LBL stack == the oracle, bitwise."""
    import numpy as np
    import paper_2404_19331_b200 as fcm
    from oracle import network as onet
    from paper_2404_19331_b200.network import Network, model_json
    plan = fcm.plan(model_json(net, "s8", 2))
    assert plan["totals"]["fused_pairs"] > 0
    a = Network(net, "s8", 2, plan)
    a.run()
    b = Network(net, "s8", 2, _lbl_plan(plan))
    b.run()
    torch.cuda.synchronize()
    assert torch.equal(a.out.cpu(), b.out.cpu())
    want = onet.forward(net, "s8", 0, 1)
    np.testing.assert_array_equal(a.out[:1].cpu().numpy().astype(np.int64), want)


@pytest.mark.parametrize("net", ["xception", "ceit_leff", "cmt_irffn", "proxylessnas_gpu"])
def test_fusion_case_networks_bf16_entries_match_oracle(net):
    """bf16: every entry of the planned (fused) stack -- FCM or LBL -- matches the oracle applied
    to that entry's own input, element-wise within the R10 tolerance."""
    import paper_2404_19331_b200 as fcm
    from oracle import network as onet
    from paper_2404_19331_b200.network import Network, model_json
    from tests.cases import as_np, compare, oracle_entry
    plan = fcm.plan(model_json(net, "bf16", 3))
    assert plan["totals"]["fused_pairs"] > 0
    a = Network(net, "bf16", 3, plan)
    a.run()
    torch.cuda.synchronize()
    prm = onet.params(net, "bf16")
    fused = 0
    for e, x, y, r in zip(a.entries, a.inputs, a.outputs, a.residuals):
        ref, mag = oracle_entry(e, a.layers, prm, as_np(x, "bf16"), "bf16", None if r is None else as_np(r, "bf16"))
        compare(as_np(y, "bf16"), ref, mag, "bf16", f"{net} {e['op']} {e['layers']}")
        fused += len(e["layers"]) == 2
    assert fused > 0

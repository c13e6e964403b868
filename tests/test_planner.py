"""fcm_plan (C++, libfcm.so) vs the planner oracle (oracle/planner.py), on CPU.

paper mode: identical entries (layers, FCM kind, Eq. GMA bytes, argmin tile) on every network.
b200 mode: every candidate's HBM bytes, exact L2->SM bytes and MACs re-derived by the oracle at
the reported tile; predicted times recomputed; the fuse rule and the chain DP re-run.
"""
import pytest

from oracle import planner as op
from oracle.counting import dw_exact, dwpw_exact, pwdw_exact
from paper_2404_19331_b200.network import model_json

CASES = [("single_dwpw", "f32", 1), ("single_dwpw", "s8", 1), ("mobilenet_v1", "s8", 64), ("mobilenet_v1", "bf16", 1),
         ("mobilenet_v2", "bf16", 256), ("mobilenet_v2", "bf16", 1), ("efficientnet_b0", "s8", 256),
         ("efficientnet_b0", "s8", 32), ("cvt13", "bf16", 512),
         ("xception", "bf16", 64), ("xception", "s8", 1), ("ceit_leff", "bf16", 256), ("cmt_irffn", "s8", 64),
         ("cmt_irffn", "bf16", 1),
         ("proxylessnas_gpu", "bf16", 64), ("proxylessnas_gpu", "s8", 1)]


@pytest.fixture(scope="module")
def fcm():
    from paper_2404_19331_b200 import build
    build.build()
    import paper_2404_19331_b200 as m
    return m


@pytest.mark.parametrize("net,dt,batch", CASES)
def test_paper_mode_matches_oracle(fcm, net, dt, batch):
    m = model_json(net, dt, batch, "paper")
    got = fcm.plan(m)["entries"]
    want = op.plan_paper(m)
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert g["layers"] == w["layers"]
        assert g["kind"] == w["kind"]
        assert g["gma_bytes"] == w["gma_bytes"]
        assert g["paper_tile"] == w["paper_tile"]


@pytest.mark.parametrize("net,dt,batch", CASES)
def test_b200_mode_candidates_and_decisions(fcm, net, dt, batch):
    """b200 mode: every candidate's compulsory HBM bytes, exact L2->SM bytes and MACs are
    re-derived by the oracle from the tile the candidate reports; the fuse rule (strict)
    and the chain DP are re-run on the library's own predicted times. (The time model is
    checked against measured kernel times in test_planner_time_model.py, not here.)"""
    m = model_json(net, dt, batch, "b200")
    p = fcm.plan(m)
    layers = {l["id"]: l for l in m["layers"]}
    order = [l["id"] for l in m["layers"]]
    lbl_cost, fcm_cost = {}, {}
    for c in p["candidates"]["lbl"] + p["candidates"]["fcm"]:
        ls = [layers[i] for i in c["layers"]]
        kern = c["op"] if len(ls) == 1 else ("dwpw" if ls[0]["kind"] == "dw" else "pwdw")
        want = op.b200_numbers(kern, ls, batch, dt, c["tile"])
        for k, v in want.items():
            assert c[k] == v, (c["layers"], k, c[k], v)
        assert c["pred_us"] > 0
        if len(ls) == 1:
            lbl_cost[c["layers"][0]] = c["pred_us"]
        else:
            accepted = c["pred_us"] < lbl_cost[c["layers"][0]] + lbl_cost[c["layers"][1]]
            assert c["accepted"] == accepted
            if accepted:
                fcm_cost[order.index(c["layers"][1])] = c["pred_us"]
    n = len(order)
    sel = op.chain_dp(n, [lbl_cost[i] for i in order], [fcm_cost.get(i) for i in range(n)])
    assert [e["layers"] for e in p["entries"]] == [[order[j] for j in e] for e in sel]
    assert p["totals"]["dram_bytes"] == sum(e["dram_bytes"] for e in p["entries"])


@pytest.mark.parametrize("gpu", ["gtx1660", "rtxa4000", "orin"])
def test_paper_mode_on_the_papers_gpus_matches_oracle(fcm, gpu):
    """Paper mode parameterised with Table 1's GPUs (RTX A4000 with its real 48 SMs,
    reading R22) equals the oracle on the paper's four end-to-end CNNs."""
    g = op.PAPER_GPUS[gpu]
    for net in ("mobilenet_v1", "mobilenet_v2", "xception", "proxylessnas_gpu"):
        m = model_json(net, "f32", 1, "paper")
        got = fcm.plan(m, g)["entries"]
        want = op.plan_paper(m, g)
        assert [(e["layers"], e["kind"], e["gma_bytes"], e["paper_tile"]) for e in got] == \
               [(e["layers"], e["kind"], e["gma_bytes"], e["paper_tile"]) for e in want]


def test_units_reduce_to_pinned_counters():
    """The batched unit counters with N=1, nb=1 equal the pinned per-image exact counters."""
    d = {"kind": "dw", "h": 13, "w": 11, "c": 40, "k": 3, "stride": 2, "pads": [1, 1, 1, 1]}
    u = op.units("dw", 1, d, 40, 40, 1, 3, 4, 1)
    e = dw_exact(13, 11, 40, 3, 2, (1,) * 4, 3, 4, 16)
    assert (u["ifm"], u["w"], u["ofm"]) == (e["ifm"], e["w"], e["ofm"])
    u = op.units("dwpw", 1, d, 40, 24, 1, 3, 4, 2)  # 24 channels in slices of 16: 2 splits
    e = dwpw_exact(13, 11, 40, 24, 3, 2, (1,) * 4, 3, 4, 16)
    assert (u["ifm"], u["w"], u["ofm"]) == (e["ifm"], e["w"], e["ofm"])
    u = op.units("pwdw", 1, d, 24, 40, 1, 3, 4, 3)  # 40 channels in slices of 16: 3 splits
    e = pwdw_exact(13, 11, 24, 40, 3, 2, (1,) * 4, 3, 4, 16)
    assert (u["ifm"], u["w"], u["ofm"]) == (e["ifm"], e["w"], e["ofm"])
    assert (u["halo"] - 13 * 11 * 40) * 24 == e["redundant_macs"]
    # batching: nb images per unit share the weight loads but not the activations
    u1 = op.units("dwpw", 4, d, 40, 24, 1, 3, 4, 2)
    u2 = op.units("dwpw", 4, d, 40, 24, 2, 3, 4, 2)
    e = dwpw_exact(13, 11, 40, 24, 3, 2, (1,) * 4, 3, 4, 16)
    assert u1["ifm"] == u2["ifm"] == 4 * e["ifm"] and u2["w"] * 2 == u1["w"]


def test_plan_rejects_bad_models(fcm):
    from paper_2404_19331_b200._lib import FcmError
    with pytest.raises(FcmError):
        fcm.plan({"dtype": "bf16", "batch": 1, "layers": []})
    with pytest.raises(FcmError):
        fcm.plan({"dtype": "bf16", "batch": 1, "layers": [
            {"id": "a", "kind": "pw", "h": 4, "w": 4, "c_in": 8, "c_out": 16},
            {"id": "b", "kind": "dw", "h": 4, "w": 4, "c": 8, "k": 3, "stride": 1}]})  # 16 != 8
    with pytest.raises(FcmError):
        fcm.plan("{not json")


def test_mobilenet_v2_fuses_every_block_and_saves_bytes(fcm):
    p = fcm.plan(model_json("mobilenet_v2", "bf16", 256, shortcuts=False))
    assert p["totals"]["fused_pairs"] == 17
    # compulsory bytes: 6605.1 MB LBL -> 2774.1 MB fused
    assert p["totals"]["lbl_dram_bytes"] == 6605130944
    assert p["totals"]["dram_bytes"] == 2774092992


@pytest.mark.parametrize("dt", ["bf16", "s8"])
def test_dwpw_tiles_respect_mma_rows_and_tmem(fcm, dt):
    # the bf16/f16 3x3 pair core takes tiles of up to 256 pixels (two M=128 MMA row blocks) when
    # 2 x 2 x C_out fits 512 TMEM columns; every other DWPW tile stays within one 128-row block
    p = fcm.plan(model_json("mobilenet_v2", dt, 256))
    net = {l["id"]: l for l in model_json("mobilenet_v2", dt, 256)["layers"]}
    big = 0
    for c in p["candidates"]["fcm"]:
        if c["op"] != "dwpw":
            continue
        t = c["tile"]
        px = t["tile_n"] * t["tile_h"] * t["tile_w"]
        cout = net[c["layers"][1]]["c_out"]
        limit = 256 if (dt == "bf16" and cout <= 128) else 128
        assert 0 < px <= limit, (c["layers"], t)
        big += px > 128
    assert (big > 0) == (dt == "bf16")

"""Host-side checks of the synthetic network tables (synth/networks.py) and the plan-refinement
tile lists (CPU only).

The tables carry only shapes, so what pins them is shape continuity (each chained block reads
exactly the previous block's output), the public architectures' layer counts and widths, and the
SURVEY §8(d) / Appendix A byte totals for the BASELINE configs.
"""
import pytest

from synth.networks import NETWORKS, block_source, layer_ids


def _out(l):
    if l["kind"] == "dw":
        ho = (l["h"] + 2 * (l["k"] // 2) - l["k"]) // l["stride"] + 1
        return ho, l["c"]
    return l["h"], l["c_out"]


def _in(l):
    return l["h"], (l["c"] if l["kind"] == "dw" else l["c_in"])


@pytest.mark.parametrize("net", sorted(NETWORKS))
def test_layers_chain_within_blocks_and_across_chained_blocks(net):
    blocks = NETWORKS[net]()
    for bi, b in enumerate(blocks):
        for a, c in zip(b, b[1:]):
            assert _out(a) == _in(c), (net, bi)
        kind, role = block_source(net, blocks, bi)
        if kind == "chain" and bi > 0:
            assert _out(blocks[bi - 1][-1]) == _in(b[0]), (net, bi)
        if kind == "stage":
            assert role.startswith(net + "/")
    for _, _, l in layer_ids(blocks):
        c = l["c"] if l["kind"] == "dw" else l["c_in"]
        assert c % 4 == 0 and (l["kind"] == "dw" or l["c_out"] % 4 == 0)


def test_fusion_case_network_shapes():
    # Xception: 34 separable convs (entry 6, middle 8 x 3, exit 4), 728 wide in the middle flow
    xc = NETWORKS["xception"]()
    assert len(xc) == 34 and sum(1 for b in xc if b[1]["c_in"] == b[1]["c_out"] == 728) == 26
    assert xc[-1][1]["c_out"] == 2048 and xc[0][0]["h"] == 147
    # ProxylessNAS-GPU: 15 MBConv + final PW 432 -> 1728, DW kernels 3/5/7
    px = NETWORKS["proxylessnas_gpu"]()
    assert len(px) == 16 and px[-1][0]["c_out"] == 1728
    assert {l["k"] for b in px for l in b if l["kind"] == "dw"} == {3, 5, 7}
    # CeiT-T LeFF: 12 x (192 -> 768 -> 192) on 14x14; CMT-S IRFFN: 3/3/16/3 blocks, expansion 4
    ce = NETWORKS["ceit_leff"]()
    assert len(ce) == 12 and all(b[0]["c_out"] == 4 * b[0]["c_in"] == 768 for b in ce)
    cm = NETWORKS["cmt_irffn"]()
    assert [sum(1 for b in cm if b[0]["h"] == h) for h in (56, 28, 14, 7)] == [3, 3, 16, 3]
    assert all(b[0]["c_out"] == 4 * b[0]["c_in"] and b[2]["c_out"] == b[0]["c_in"] for b in cm)


def test_mobilenet_v2_compulsory_bytes_match_survey_appendix():
    # MobileNetV2 bf16 b256, LBL 6605 MB (the per-layer §8(d) formulas)
    b, n = 2, 256
    tot = 0
    for _, _, l in layer_ids(NETWORKS["mobilenet_v2"]()):
        if l["kind"] == "dw":
            ho, _ = _out(l)
            tot += b * (n * (l["h"] * l["w"] * l["c"] + ho * ho * l["c"]) + l["k"] ** 2 * l["c"])
        else:
            tot += b * (n * l["h"] * l["w"] * (l["c_in"] + l["c_out"]) + l["c_in"] * l["c_out"])
    assert round(tot / 1e6) == 6605


def test_dw_tile_alternatives_fit_the_kernel_limits():
    from paper_2404_19331_b200.autotune import dw_tile_alternatives
    base = {"tile_n": 1, "tile_h": 8, "tile_w": 16, "n_split": 0}
    for (ho, k, s, c, dt) in [(56, 3, 1, 128, "s8"), (7, 7, 1, 1024, "bf16"), (112, 3, 2, 32, "f32"), (14, 5, 1, 672, "s8")]:
        alts = dw_tile_alternatives(base, ho, ho, k, s, c, dt)
        assert alts[0] == base and len({(t["tile_h"], t["tile_w"]) for t in alts}) == len(alts)
        for t in alts[1:]:
            assert 1 <= t["tile_h"] <= ho and 1 <= t["tile_w"] <= ho
            assert (t["tile_h"] - 1) * s + k <= 256 and (t["tile_w"] - 1) * s + k <= 256

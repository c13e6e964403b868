"""Pins for oracle/counting.py: the paper's worked two-mapping example, SPEC's
verbatim evaluations of Eq. 1-4, brute-force element-set enumeration of the exact counters,
and the c13 closed form."""
import itertools
import json
import os
import random

import pytest

from oracle import counting as cnt

GOLD = os.path.join(os.path.dirname(__file__), "golden")
S = json.load(open(os.path.join(GOLD, "spec_equation_values.json")))


def test_eq1_overlap():
    assert cnt.overlap(6, 6, 3, 3, 3, 3, 1) == S["overlap_6x6_t3x3_f3_s1"]
    assert cnt.overlap(6, 6, 6, 6, 3, 3, 1) == 0
    assert cnt.overlap(6, 6, 2, 2, 1, 1, 1) == 0
    assert cnt.overlap(6, 6, 2, 2, 1, 1, 2) == 0  # (F-S) clamped at 0


def test_eq3_dw_gma():
    ovl = cnt.overlap(6, 6, 3, 3, 3, 3, 1)
    assert cnt.dw_gma(4, ovl, 144, 144, 36, 9, 36) == S["dw_gma_6x6x4_f3_s1_tiled_3x3"]
    assert cnt.dw_gma(4, 0, 144, 144, 36, 36, 36) == S["dw_gma_6x6x4_f3_s1_single"]


def test_eq2_pw_gma():
    assert cnt.pw_gma(128, 256, 128, 128, 256) == S["pw_gma_4x4x8_to16_single"]
    assert cnt.pw_gma(128, 256, 128, 64, 128) == S["pw_gma_4x4x8_to16_two_partitions"]
    assert 1 * cnt.pw_gma(128, 256, 128, 128, 256) == S["pw_gma_4x4x8_to16_single_int8_bytes"]


def test_eq4_pwdw_gma():
    args = dict(pw_d=4, dw_ovl=0, pw_ifm=144, pw_w=32, pw_wt=32, dw_w=72, dw_wt=72, dw_ofm=288, dw_ofmt=288,
                dw_ofm_hw=36, dw_ofmt_hw=36)
    assert cnt.pwdw_gma(**args, mode="paper") == S["pwdw_gma_6x6x4_to8_f3_single_paper"]
    assert cnt.pwdw_gma(**args, mode="consistent") == S["pwdw_gma_6x6x4_to8_f3_single_consistent"]


def test_paper_two_mapping_example():
    """P:597-601. IFM + weights only (the example excludes the OFM store)."""
    g = json.load(open(os.path.join(GOLD, "paper_two_mapping.json")))
    ifm, w, ofm = 6 * 6 * 4, 4 * 4, 6 * 6 * 4
    # Mapping1: weights partitioned over 2 SMs (2 filters each), full spatial tile
    m1 = cnt.pw_exact(6, 6, 4, 4, 6, 6, 2)
    assert m1["ifm"] + m1["w"] == g["mapping1_ifm_plus_weights"]
    # Mapping2: spatial halves, all filters per SM
    m2 = cnt.pw_exact(6, 6, 4, 4, 3, 6, 4)
    assert m2["ifm"] + m2["w"] == g["mapping2_ifm_plus_weights"]
    assert round(100 * (1 - (m2["ifm"] + m2["w"]) / (m1["ifm"] + m1["w"]))) == g["saving_percent"]
    # Eq. 2 under the OS-LWS reading (OFM tile = spatial tile x ALL channels) gives the same
    assert cnt.pw_gma(ifm, ofm, w, 8, 144) - ofm == g["mapping1_ifm_plus_weights"]
    assert cnt.pw_gma(ifm, ofm, w, 16, 72) - ofm == g["mapping2_ifm_plus_weights"]
    # max weight reuse: MACs a weight serves inside one SM = spatial pixels it slides over
    assert 6 * 6 == g["mapping1_max_weight_reuse"] and 3 * 6 == g["mapping2_max_weight_reuse"]


def test_exact_counts_on_spec_examples():
    e = cnt.dw_exact(6, 6, 4, 3, 1, (1,) * 4, 3, 3, 4)
    assert e["total"] == S["dw_exact_6x6x4_f3_s1_tiled_3x3"]
    assert e["ifm"] - 144 == 4 * S["overlap_exact_extra_loads_per_channel"]
    assert cnt.pw_exact(4, 4, 8, 16, 4, 4, 8)["total"] == S["pw_exact_4x4x8_to16_two_partitions"]
    r = cnt.pwdw_exact(6, 6, 4, 8, 3, 1, (1,) * 4, 3, 3, 8)
    assert r["redundant_macs"] == S["pwdw_r_redundancy_exact_num"]
    ratio = cnt.redundancy_ratio(6, 6, 4, 8, 3, 1, (1,) * 4, 3, 3, 8)
    assert ratio == pytest.approx(S["pwdw_r_redundancy_exact_num"] / S["pwdw_r_redundancy_exact_den"])
    # Eq.-based ratio: Overlap * depth * per-element MACs
    red_eq = cnt.overlap(6, 6, 3, 3, 3, 3, 1) * 8 * 4
    assert red_eq / (1152 + 2592 + red_eq) == pytest.approx(S["pwdw_r_redundancy_eq_based"], abs=5e-4)


def _brute_dw_loads(h, w, c, k, s, pads, th, tw, td):
    """Element-set enumeration: for every unit, the set of in-image input elements touched."""
    pt, pl, pb, pr = pads
    ho, wo = (h + pt + pb - k) // s + 1, (w + pl + pr - k) // s + 1
    total = 0
    for y0 in range(0, ho, th):
        for x0 in range(0, wo, tw):
            for c0 in range(0, c, td):
                need = set()
                for y in range(y0, min(y0 + th, ho)):
                    for x in range(x0, min(x0 + tw, wo)):
                        for cc in range(c0, min(c0 + td, c)):
                            for i, j in itertools.product(range(k), range(k)):
                                yy, xx = y * s - pt + i, x * s - pl + j
                                if 0 <= yy < h and 0 <= xx < w:
                                    need.add((yy, xx, cc))
                total += len(need)
    return total


def test_exact_dw_counter_matches_element_enumeration():
    r = random.Random(7)
    for _ in range(60):
        k = r.choice([1, 3, 5])
        s = r.choice([1, 2])
        p = r.choice([0, k // 2])
        h, w, c = r.randint(k, 11), r.randint(k, 11), r.randint(1, 4)
        ho, wo = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
        th, tw, td = r.randint(1, ho), r.randint(1, wo), r.randint(1, c)
        assert cnt.dw_exact(h, w, c, k, s, (p,) * 4, th, tw, td)["ifm"] == \
            _brute_dw_loads(h, w, c, k, s, (p,) * 4, th, tw, td)


def test_exact_closed_form_c13():
    """Evenly dividing tiles, pad k//2: per-channel loads = (H+(nH-1)(k-s))(W+(nW-1)(k-s))."""
    r = random.Random(9)
    for _ in range(300):
        k, s = r.choice([(3, 1), (5, 1), (3, 2), (5, 2)])
        nh, nw = r.randint(1, 5), r.randint(1, 5)
        lo = -(-k // s)  # tiles at least one filter wide: halos clip only at the image edge
        th, tw = r.randint(lo, 6), r.randint(lo, 6)
        h, w = nh * th * s, nw * tw * s
        got = cnt.dw_exact(h, w, 1, k, s, (k // 2,) * 4, th, tw, 1)["ifm"]
        assert got == (h + (nh - 1) * (k - s)) * (w + (nw - 1) * (k - s))
        if s == 1:  # Eq. 1 misses only the tile-corner term
            assert got == h * w + cnt.overlap(h, w, th, tw, k, k, s) + (nh - 1) * (nw - 1) * (k - s) ** 2


def test_single_tile_equals_compulsory():
    """with one all-covering tile every estimator is IFM + W + OFM."""
    assert cnt.dw_exact(9, 9, 5, 3, 1, (1,) * 4, 9, 9, 5)["total"] == 81 * 5 * 2 + 45
    assert cnt.pw_exact(4, 4, 8, 16, 4, 4, 16)["total"] == 128 + 256 + 128
    assert cnt.dwpw_exact(7, 7, 8, 12, 3, 1, (1,) * 4, 7, 7, 12)["total"] == \
        cnt.compulsory("dwpw", 1, 7, 7, 8, 12, 3, 1)
    assert cnt.pwdw_exact(7, 7, 8, 12, 3, 1, (1,) * 4, 7, 7, 12)["total"] == \
        cnt.compulsory("pwdw", 1, 7, 7, 8, 12, 3, 1)


def test_fused_saving_is_twice_intermediate():
    """Compulsory bytes: unfused DW+PW minus fused DWPW = 2 x |T| (write + re-read)."""
    n, h, c_in, c_out = 3, 14, 16, 32
    lbl = cnt.compulsory("dw", n, h, h, c_in, c_in, 3, 1) + cnt.compulsory("pw", n, h, h, c_in, c_out)
    assert lbl - cnt.compulsory("dwpw", n, h, h, c_in, c_out, 3, 1) == 2 * n * h * h * c_in


def test_decision_rule_strict():
    assert cnt.fused_wins(9, 10) and not cnt.fused_wins(10, 10)

"""FusePlanner oracle (TEST INFRASTRUCTURE -- see oracle/__init__).

paper mode: the paper's procedure written out plainly: for every layer, minimise
  Eq. 2 / Eq. 3 over the tile grid subject to the two constraints (on-chip capacity, #OFM tiles
  >= #SMs -- waived when unsatisfiable, reading R17); for every adjacent single-consumer pair,
  minimise the FCM equation (Eq. 4 for PW->DW, the constructed DWPW equation for DW->PW); keep a
  pair iff FCM < LBL sum; choose non-overlapping pairs by a chain DP.
  Every GMA value comes from the pinned equation functions of oracle/counting.py (Eq. 1
  overlap, Eq. 2 pw_gma, Eq. 3 dw_gma, Eq. 4 pwdw_gma, the constructed dwpw_gma); only the grid
  and the two constraints are written here. A layer whose grid is empty (no tile fits on chip)
  is left untiled: one tile, GMA = IFM + W + OFM (the single-tile closed form).
b200 mode: re-derive, from the candidate's reported tile (images x rows x cols per tile, number
  of channel splits), its compulsory HBM bytes (counting.compulsory), its exact L2->SM element
  counts (exact unit enumeration) and its MACs; re-run the decision rule and the chain
  DP on the library's reported times. The time model itself is not mirrored here: it
  is checked against measured kernel times (tests/test_planner_time_model.py).
Grid (reading R18): spatial {1,2,4,8,16,32,64, n, divisors of n <= 64} within [1, n]; depth
  {multiples of 32 <= D} U {D}; enumeration order (td, th, tw), first minimum wins; for PW->DW a
  full-map tile (PWDW, no redundancy) wins ties against PWDW_R.
"""
from __future__ import annotations

from math import ceil

from oracle.counting import compulsory, dw_gma, dwpw_gma, overlap, pw_gma, pwdw_gma, tiles_1d, touched

ESZ = {"f32": 4, "bf16": 2, "f16": 2, "s8": 1}


def cand(n):
    c = {1, 2, 4, 8, 16, 32, 64, n} | {d for d in range(1, min(n, 64) + 1) if n % d == 0}
    return sorted(v for v in c if 1 <= v <= n)


def dcand(d):
    return sorted({d} | set(range(32, d + 1, 32)))


def out_hw(l):
    if l["kind"] == "pw":
        return l["h"], l["w"]
    pt, pl, pb, pr = l.get("pads", [l["k"] // 2] * 4)
    return (l["h"] + pt + pb - l["k"]) // l["stride"] + 1, (l["w"] + pl + pr - l["k"]) // l["stride"] + 1


def _search(fn, sms):
    """#OFM tiles >= #SMs, waived when unsatisfiable (reading R17)."""
    best = fn(sms)
    return best if best is not None else fn(1)


def paper_dw(l, N, b, sms, smem):
    H, W, C, k, s = l["h"], l["w"], l["c"], l["k"], l["stride"]
    Ho, Wo = out_hw(l)

    def run(min_tiles):
        best = None
        for td in dcand(C):
            for th in cand(Ho):
                for tw in cand(Wo):
                    if (th * tw * td) % 32:
                        continue
                    if N * ceil(Ho / th) * ceil(Wo / tw) * ceil(C / td) < min_tiles:
                        continue
                    thi, twi = min((th - 1) * s + k, H), min((tw - 1) * s + k, W)
                    if (thi * twi * td + th * tw * td + k * k * td) * b > smem:
                        continue
                    ov = N * overlap(H, W, th * s, tw * s, k, k, s)      # Eq. 1, every image
                    gma = dw_gma(C, ov, N * H * W * C, N * Ho * Wo * C, N * Ho * Wo, th * tw, k * k * C)  # Eq. 3
                    if best is None or gma < best[0]:
                        best = (gma, th, tw, td, "dw")
        return best
    return _search(run, sms) or (N * H * W * C + k * k * C + N * Ho * Wo * C, Ho, Wo, C, "dw")


def paper_pw(l, N, b, sms, smem):
    H, W, Ci, Co = l["h"], l["w"], l["c_in"], l["c_out"]

    def run(min_tiles):
        best = None
        for td in dcand(Co):
            for th in cand(H):
                for tw in cand(W):
                    if (th * tw * td) % 32:
                        continue
                    if N * ceil(H / th) * ceil(W / tw) * ceil(Co / td) < min_tiles:
                        continue
                    if (th * tw * Ci + th * tw * td + td * Ci) * b > smem:
                        continue
                    gma = pw_gma(N * H * W * Ci, N * H * W * Co, Ci * Co, td * Ci, th * tw * td)  # Eq. 2
                    if best is None or gma < best[0]:
                        best = (gma, th, tw, td, "pw")
        return best
    return _search(run, sms) or (N * H * W * Ci + Ci * Co + N * H * W * Co, H, W, Co, "pw")


def paper_pwdw(p, d, N, b, sms, smem):
    Ci, Cm = p["c_in"], p["c_out"]
    H, W, k, s = d["h"], d["w"], d["k"], d["stride"]
    Ho, Wo = out_hw(d)

    def run(min_tiles):
        best = None
        for td in dcand(Cm):
            for th in cand(Ho):
                for tw in cand(Wo):
                    if (th * tw * td) % 32:
                        continue
                    if N * ceil(Ho / th) * ceil(Wo / tw) * ceil(Cm / td) < min_tiles:
                        continue
                    thi, twi = min((th - 1) * s + k, H), min((tw - 1) * s + k, W)
                    if (thi * twi * Ci + th * tw * td + td * Ci + k * k * td + thi * twi * td) * b > smem:
                        continue
                    ov = N * overlap(H, W, th * s, tw * s, k, k, s)
                    gma = pwdw_gma(Ci, ov, N * H * W * Ci, Ci * Cm, td * Ci, k * k * Cm, k * k * td,
                                   N * Ho * Wo * Cm, th * tw * td, N * Ho * Wo, th * tw)   # Eq. 4 + DwOFM (R15)
                    kind = "pwdw" if (th == Ho and tw == Wo) else "pwdw_r"
                    if best is None or gma < best[0] or (gma == best[0] and kind == "pwdw" and best[4] == "pwdw_r"):
                        best = (gma, th, tw, td, kind)
        return best
    return _search(run, sms)


def paper_dwpw(d, p, N, b, sms, smem):
    Ci, Co = d["c"], p["c_out"]
    H, W, k, s = d["h"], d["w"], d["k"], d["stride"]
    Ho, Wo = out_hw(d)

    def run(min_tiles):
        best = None
        for td in dcand(Co):
            for th in cand(Ho):
                for tw in cand(Wo):
                    if (th * tw * td) % 32:
                        continue
                    if N * ceil(Ho / th) * ceil(Wo / tw) * ceil(Co / td) < min_tiles:
                        continue
                    thi, twi = min((th - 1) * s + k, H), min((tw - 1) * s + k, W)
                    if (thi * twi * Ci + th * tw * td + k * k * Ci + Ci * td + th * tw * Ci) * b > smem:
                        continue
                    ov = N * overlap(H, W, th * s, tw * s, k, k, s)
                    gma = dwpw_gma(Ci, ov, N * H * W * Ci, k * k * Ci, Ci * Co, Ci * td, N * Ho * Wo * Co,
                                   th * tw * td, N * Ho * Wo, th * tw)   # constructed (R13)
                    if best is None or gma < best[0]:
                        best = (gma, th, tw, td, "dwpw")
        return best
    return _search(run, sms)


# ------------------------------------------------------------------ B200 byte / MAC accounting
def units(kind, N, d, c_in, c_x, nb, th, tw, ns):
    """Exact unit enumeration of a B200 kernel launch (reading R21): a unit = nb images x th x tw
    output tile x one of `ns` channel splits (of C_out for dwpw, of C_mid for pwdw; dw units
    cover every channel). Every unit loads its clipped input halo (padding is never fetched) --
    over ALL C_in channels for the fused kinds -- its weights, and stores its outputs once.
    Counts are in elements; the split widths sum to the channel count, so only `ns` matters."""
    Ho, Wo = out_hw(d)
    pt, pl = d.get("pads", [d["k"] // 2] * 4)[:2]
    k = d["k"]
    ifm = w = halo = 0
    for n0 in range(0, N, nb):
        nbe = min(nb, N - n0)
        for (y0, y1) in tiles_1d(Ho, th):
            ny = touched(y0, y1, k, d["stride"], pt, d["h"])
            for (x0, x1) in tiles_1d(Wo, tw):
                px = nbe * ny * touched(x0, x1, k, d["stride"], pl, d["w"])
                if kind == "dw":
                    ifm += px * c_in
                    w += k * k * c_in
                elif kind == "dwpw":
                    ifm += ns * px * c_in
                    w += ns * k * k * c_in + c_in * c_x
                else:
                    ifm += ns * px * c_in
                    w += c_in * c_x + k * k * c_x
                    halo += px * c_x
    return {"ifm": ifm, "w": w, "ofm": N * Ho * Wo * (c_in if kind == "dw" else c_x), "halo": halo}


def pw_units(M, ci, co, bm, ns):
    """PW launch: row blocks of bm pixels x ns column splits; each block reads its A rows once
    per split and the weights once per row block."""
    return {"ifm": ns * M * ci, "w": ceil(M / bm) * co * ci, "ofm": M * co}


def b200_numbers(op, layers, N, dtype, tile):
    """Compulsory HBM bytes, exact L2->SM bytes and MACs of one candidate at the
    tile it reports (tile_n, tile_h, tile_w, n_split). A last layer with a residual (shortcut)
    epilogue also reads one output-shaped tensor."""
    out = _b200_numbers(op, layers, N, dtype, tile)
    last = layers[-1]
    if last.get("residual"):
        Ho, Wo = out_hw(last)
        out["dram_bytes"] += N * Ho * Wo * last["c_out"] * ESZ[dtype]
    return out


def _b200_numbers(op, layers, N, dtype, tile):
    b = ESZ[dtype]
    nb, th, tw, ns = tile["tile_n"], tile["tile_h"], tile["tile_w"], tile["n_split"]
    if op == "dw":
        d = layers[0]
        Ho, Wo = out_hw(d)
        u = units("dw", N, d, d["c"], d["c"], 1, th, tw, 1)
        return dict(dram_bytes=compulsory("dw", N, d["h"], d["w"], d["c"], d["c"], d["k"], d["stride"]) * b,
                    l2_bytes=(u["ifm"] + u["w"] + u["ofm"]) * b,
                    dw_macs=N * Ho * Wo * d["c"] * d["k"] ** 2, pw_macs=0, redundant_macs=0)
    if op == "pw":
        p = layers[0]
        M = N * p["h"] * p["w"]
        ci, co = p["c_in"], p["c_out"]
        u = pw_units(M, ci, co, th, ns)
        return dict(dram_bytes=compulsory("pw", N, p["h"], p["w"], ci, co) * b,
                    l2_bytes=(u["ifm"] + u["w"] + u["ofm"]) * b, dw_macs=0, pw_macs=M * ci * co, redundant_macs=0)
    if op == "dwpw":
        d, p = layers
        Ho, Wo = out_hw(d)
        ci, co = d["c"], p["c_out"]
        u = units("dwpw", N, d, ci, co, nb, th, tw, ns)
        return dict(dram_bytes=compulsory("dwpw", N, d["h"], d["w"], ci, co, d["k"], d["stride"]) * b,
                    l2_bytes=(u["ifm"] + u["w"] + u["ofm"]) * b,
                    dw_macs=N * Ho * Wo * ci * d["k"] ** 2 * ns, pw_macs=N * Ho * Wo * ci * co, redundant_macs=0)
    p, d = layers
    Ho, Wo = out_hw(d)
    ci, cm = p["c_in"], p["c_out"]
    u = units("pwdw", N, d, ci, cm, nb, th, tw, ns)
    return dict(dram_bytes=compulsory("pwdw", N, d["h"], d["w"], ci, cm, d["k"], d["stride"]) * b,
                l2_bytes=(u["ifm"] + u["w"] + u["ofm"]) * b, dw_macs=N * Ho * Wo * cm * d["k"] ** 2,
                pw_macs=u["halo"] * ci, redundant_macs=(u["halo"] - N * d["h"] * d["w"] * cm) * ci)


def chain_dp(n, lbl_cost, fcm_cost):
    """dp[i] = best cost of layers [0, i); fcm_cost[i] = cost of fusing (i-1, i) or None.
    A fusion wins ties (later fusion preferred). Returns the entry list [(i0,), (i0, i1), ...]."""
    dp, take = [0.0] * (n + 1), [0] * (n + 1)
    for i in range(1, n + 1):
        dp[i], take[i] = dp[i - 1] + lbl_cost[i - 1], 1
        if i >= 2 and fcm_cost[i - 1] is not None:
            v = dp[i - 2] + fcm_cost[i - 1]
            if v <= dp[i]:
                dp[i], take[i] = v, 2
    out, i = [], n
    while i > 0:
        if take[i] == 2:
            out.append((i - 2, i - 1))
            i -= 2
        else:
            out.append((i - 1,))
            i -= 1
    return out[::-1]


def fusable(layers, edges):
    """fus[i] True iff (i-1 -> i) is an edge, i-1 has one consumer and i one producer, and the
    kinds admit an FCM (DW->PW: DWPW; PW->DW: PWDW/PWDW_R)."""
    n = len(layers)
    ids = [l["id"] for l in layers]
    if edges is None:
        edges = [[ids[i - 1], ids[i]] for i in range(1, n)]
    outd, ind = {l["id"]: l.get("extra_consumers", 0) for l in layers}, {i: 0 for i in ids}  # + residual readers
    es = set()
    for a, c in edges:
        outd[a] += 1
        ind[c] += 1
        es.add((a, c))
    fus = [False] * n
    for i in range(1, n):
        a, c = layers[i - 1], layers[i]
        if (a["id"], c["id"]) in es and outd[a["id"]] == 1 and ind[c["id"]] == 1 and a["kind"] != c["kind"]:
            fus[i] = True
    return fus


PAPER_GPU = dict(num_sms=148, smem_bytes=232448)  # B200: 148 SMs, 227 KB shared memory per CTA
# Table 1: #SMs and L1 per SM of the paper's GPUs. The RTX A4000's printed "128"
# SMs is garbled (6144 cores / 128 per Ampere SM = 48, reading R22).
PAPER_GPUS = {"gtx1660": dict(num_sms=22, smem_bytes=96 * 1024),
              "rtxa4000": dict(num_sms=48, smem_bytes=128 * 1024),
              "orin": dict(num_sms=16, smem_bytes=192 * 1024)}


def plan_paper(model, gpu=None):
    g = dict(PAPER_GPU, **(gpu or {}))
    b, N = ESZ[model["dtype"]], model["batch"]
    L = model["layers"]
    sms, smem = g["num_sms"], g["smem_bytes"]
    lbl = [paper_dw(l, N, b, sms, smem) if l["kind"] == "dw" else paper_pw(l, N, b, sms, smem) for l in L]
    fus = fusable(L, model.get("edges"))
    fc = [None] * len(L)
    for i in range(1, len(L)):
        if not fus[i]:
            continue
        a, c = L[i - 1], L[i]
        r = paper_dwpw(a, c, N, b, sms, smem) if a["kind"] == "dw" else paper_pwdw(a, c, N, b, sms, smem)
        if r is not None and r[0] < lbl[i - 1][0] + lbl[i][0]:
            fc[i] = r
    sel = chain_dp(len(L), [x[0] for x in lbl], [None if x is None else x[0] for x in fc])
    return [dict(layers=[L[j]["id"] for j in e], kind=(lbl[e[0]][4] if len(e) == 1 else fc[e[1]][4]),
                 gma_bytes=(lbl[e[0]][0] if len(e) == 1 else fc[e[1]][0]) * b,
                 paper_tile=dict(zip(("th", "tw", "td"), (lbl[e[0]] if len(e) == 1 else fc[e[1]])[1:4])))
            for e in sel]

"""FusePlanner oracle (TEST INFRASTRUCTURE -- see oracle/__init__).

paper mode: the paper's procedure written out plainly: for every layer, minimise
  Eq. 2 / Eq. 3 over the tile grid subject to the two constraints (on-chip capacity, #OFM tiles
  >= #SMs -- waived when unsatisfiable, reading R17); for every adjacent single-consumer pair,
  minimise the FCM equation (Eq. 4 for PW->DW, the constructed DWPW equation for DW->PW); keep a
  pair iff FCM < LBL sum; choose non-overlapping pairs by a chain DP.
b200 mode: re-derive every candidate the library reports -- compulsory HBM bytes, exact unit
  counts at the reported tile (counting.*_units), MACs and the predicted time -- and re-run the
  decision + DP from those numbers.
Grid (reading R18): spatial {1,2,4,8,16,32,64, n, divisors of n <= 64} within [1, n]; depth
  {multiples of 32 <= D} U {D}; enumeration order (td, th, tw), first minimum wins; for PW->DW a
  full-map tile (PWDW, no redundancy) wins ties against PWDW_R.
"""
from __future__ import annotations

from math import ceil

from oracle.counting import overlap, tiles_1d, touched

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
                    ov = overlap(H, W, th * s, tw * s, k, k, s)          # Eq. 1
                    gma = 2 * C * N * ov + N * H * W * C + N * Ho * Wo * C + ceil(N * Ho * Wo / (th * tw)) * k * k * C
                    if best is None or gma < best[0]:                    # Eq. 3
                        best = (gma, th, tw, td, "dw")
        return best
    return _search(run, sms)


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
                    gma = ceil(Ci * Co / (td * Ci)) * N * H * W * Ci + N * H * W * Co + \
                        ceil(N * H * W * Co / (th * tw * td)) * Ci * Co    # Eq. 2
                    if best is None or gma < best[0]:
                        best = (gma, th, tw, td, "pw")
        return best
    return _search(run, sms)


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
                    ov = overlap(H, W, th * s, tw * s, k, k, s)
                    rep = max(ceil(Ci * Cm / (td * Ci)), ceil(k * k * Cm / (k * k * td)))
                    gma = (2 * Ci * N * ov + N * H * W * Ci) * rep + ceil(N * Ho * Wo * Cm / (th * tw * td)) * Ci * Cm + \
                        ceil(N * Ho * Wo / (th * tw)) * k * k * Cm + N * Ho * Wo * Cm   # Eq. 4 + store
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
                    ov = overlap(H, W, th * s, tw * s, k, k, s)
                    nw = ceil(Ci * Co / (Ci * td))
                    gma = (2 * Ci * N * ov + N * H * W * Ci) * nw + ceil(N * Ho * Wo / (th * tw)) * nw * k * k * Ci + \
                        ceil(N * Ho * Wo * Co / (th * tw * td)) * Ci * Co + N * Ho * Wo * Co
                    if best is None or gma < best[0]:
                        best = (gma, th, tw, td, "dwpw")
        return best
    return _search(run, sms)


# ------------------------------------------------------------------ B200 byte / MAC model
def units(kind, N, d, c_in, c_x, nb, th, tw, sl):
    """Exact unit enumeration: unit = nb images x th x tw output tile x channel slice `sl`."""
    Ho, Wo = out_hw(d)
    pt, pl = d.get("pads", [d["k"] // 2] * 4)[:2]
    cs = c_in if kind == "dw" else c_x
    ifm = w = halo = 0
    for n0 in range(0, N, nb):
        nbe = min(nb, N - n0)
        for (y0, y1) in tiles_1d(Ho, th):
            ny = touched(y0, y1, d["k"], d["stride"], pt, d["h"])
            for (x0, x1) in tiles_1d(Wo, tw):
                nx = touched(x0, x1, d["k"], d["stride"], pl, d["w"])
                for (c0, c1) in tiles_1d(cs, sl):
                    ce, px = c1 - c0, nbe * ny * nx
                    if kind == "dw":
                        ifm += px * ce
                        w += d["k"] ** 2 * ce
                    elif kind == "dwpw":
                        ifm += px * c_in
                        w += d["k"] ** 2 * c_in + c_in * ce
                    else:
                        ifm += px * c_in
                        w += c_in * ce + d["k"] ** 2 * ce
                        halo += px * ce
    return {"ifm": ifm, "w": w, "ofm": N * Ho * Wo * cs, "halo": halo}


def pw_units(M, ci, co, bm, bn):
    return {"ifm": ceil(co / bn) * M * ci, "w": ceil(M / bm) * co * ci, "ofm": M * co}


DEFAULT_GPU = dict(num_sms=148, smem_bytes=232448, hbm_gbs=6534.5, l2_gbs=20000.0, tc_tmacs=832.0,
                   ffma_tmacs=37.2, dw_eff=0.5, launch_us=2.0, dw_eff_i8=0.17, dw_eff_i8_fused=0.085)


def pred_us(c, dtype, g):
    hbm = c["dram_bytes"] / (g["hbm_gbs"] * 1e3)
    l2 = c["l2_bytes"] / (g["l2_gbs"] * 1e3)
    eff = (g["dw_eff_i8"] if c["op"] == "dw" else g["dw_eff_i8_fused"]) if dtype == "s8" else g["dw_eff"]
    dw = c["dw_macs"] / (g["ffma_tmacs"] * 1e6 * eff)
    tcr = g["ffma_tmacs"] if dtype == "f32" else (2.0 if dtype == "s8" else 1.0) * g["tc_tmacs"]
    pw = c["pw_macs"] / (tcr * 1e6)
    return max(max(hbm, l2), max(dw, pw)) + g["launch_us"]


def _bn(co, ns, b):
    """PW column block of the tensor-core kernels: one block padded to 16 when ns == 1, else a
    multiple of the 128-byte store chunk (128/b columns), at most 256."""
    if ns == 1:
        return (co + 15) // 16 * 16
    cpc = 128 // b
    return min((ceil(co / ns) + cpc - 1) // cpc * cpc, 256)


def _simt(dtype, b, *chans):
    """fp32 and any NHWC pitch that is not a multiple of 16 bytes run on the CUDA-core kernels."""
    return dtype == "f32" or any((c * b) % 16 for c in chans)


def b200_numbers(op, layers, N, dtype, tile):
    """Compulsory HBM bytes, exact L2->SM bytes and MACs of one candidate at its reported tile."""
    b = ESZ[dtype]
    nb, th, tw, ns = tile["tile_n"], tile["tile_h"], tile["tile_w"], tile["n_split"]
    if op == "dw":
        d = layers[0]
        Ho, Wo = out_hw(d)
        u = units("dw", N, d, d["c"], d["c"], 1, th, tw, d["c"] if (d["c"] * b) % 16 else 128 // b)
        dram = (N * (d["h"] * d["w"] * d["c"] + Ho * Wo * d["c"]) + d["k"] ** 2 * d["c"]) * b
        return dict(dram_bytes=dram, l2_bytes=(u["ifm"] + u["w"] + u["ofm"]) * b,
                    dw_macs=N * Ho * Wo * d["c"] * d["k"] ** 2, pw_macs=0, redundant_macs=0)
    if op == "pw":
        p = layers[0]
        M = N * p["h"] * p["w"]
        ci, co = p["c_in"], p["c_out"]
        bm = th
        bn = 64 if _simt(dtype, b, ci, co) else _bn(co, ns, b)
        u = pw_units(M, ci, co, bm, bn)
        return dict(dram_bytes=(M * (ci + co) + ci * co) * b, l2_bytes=(u["ifm"] + u["w"] + u["ofm"]) * b,
                    dw_macs=0, pw_macs=M * ci * co, redundant_macs=0)
    if op == "dwpw":
        d, p = layers
        Ho, Wo = out_hw(d)
        ci, co = d["c"], p["c_out"]
        bn = 64 if _simt(dtype, b, ci, co) else _bn(co, ns, b)
        u = units("dwpw", N, d, ci, co, nb, th, tw, bn)
        dram = (N * (d["h"] * d["w"] * ci + Ho * Wo * co) + d["k"] ** 2 * ci + ci * co) * b
        return dict(dram_bytes=dram, l2_bytes=(u["ifm"] + u["w"] + u["ofm"]) * b,
                    dw_macs=N * Ho * Wo * ci * d["k"] ** 2 * ns, pw_macs=N * Ho * Wo * ci * co, redundant_macs=0)
    p, d = layers
    Ho, Wo = out_hw(d)
    ci, cm = p["c_in"], p["c_out"]
    td = 32 if _simt(dtype, b, ci, cm) else 128 // b
    u = units("pwdw", N, d, ci, cm, nb, th, tw, td)
    dram = (N * (d["h"] * d["w"] * ci + Ho * Wo * cm) + ci * cm + d["k"] ** 2 * cm) * b
    return dict(dram_bytes=dram, l2_bytes=(u["ifm"] + u["w"] + u["ofm"]) * b, dw_macs=N * Ho * Wo * cm * d["k"] ** 2,
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
    outd, ind = {i: 0 for i in ids}, {i: 0 for i in ids}
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


def plan_paper(model, gpu=None):
    g = dict(DEFAULT_GPU, **(gpu or {}))
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

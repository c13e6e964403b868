"""Measured plan refinement ("measure, don't guess").

FusePlanner (fcm_plan, b200 mode) ranks options with an analytic time model. This module times
every candidate the planner reports -- each layer's LBL kernel and each admissible FCM -- on the
current GPU (CUDA events, L2-warm, the candidate's own tile) and re-runs the same decision rule
(fuse iff strictly faster) and chain DP on the measured times.
The returned plan has the planner's format; entries carry `measured_us`.
"""
from __future__ import annotations

import copy

import torch

import paper_2404_19331_b200 as fcm
from paper_2404_19331_b200.network import Network, model_json


def _time(f, reps=10):
    for _ in range(2):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def chain_dp(order, lbl, fcm_cost):
    """Same DP as planner.cpp: dp over the layer chain, a fusion (i-1, i) wins exact ties."""
    n = len(order)
    dp, take = [0.0] * (n + 1), [0] * (n + 1)
    for i in range(1, n + 1):
        dp[i], take[i] = dp[i - 1] + lbl[order[i - 1]], 1
        key = (order[i - 2], order[i - 1]) if i >= 2 else None
        if key in fcm_cost and dp[i - 2] + fcm_cost[key] <= dp[i]:
            dp[i], take[i] = dp[i - 2] + fcm_cost[key], 2
    sel, i = [], n
    while i > 0:
        if take[i] == 2:
            sel.append((order[i - 2], order[i - 1]))
            i -= 2
        else:
            sel.append((order[i - 1],))
            i -= 1
    return sel[::-1], dp[n]


def dwpw_tile_alternatives(tile, ho, wo, k, s, cout, dtype, limit=10):
    """A few DWPW output tiles besides the planner's (measured, not modelled, choice): row/column
    extents from {4, 7, 8, 14, 16, 28} that fit the MMA rows (256 for the bf16/f16 3x3 pair core
    when 2 x 2 x C_out <= 512 TMEM columns, else 128), whole-map tiles with several images."""
    mmax = 256 if (dtype in ("bf16", "f16") and k == 3 and cout <= 128) else 128
    out = [dict(tile)]
    sizes = [4, 7, 8, 14, 16, 28]
    for th in sizes:
        for tw in sizes:
            if th > ho or tw > wo or th * tw > mmax or th * tw < 32 or (s == 2 and th * tw > 128):
                continue
            out.append({"tile_n": 1, "tile_h": th, "tile_w": tw, "n_split": tile.get("n_split", 1)})
    if ho * wo <= mmax // 2:
        for nb in range(2, mmax // (ho * wo) + 1):
            out.append({"tile_n": nb, "tile_h": ho, "tile_w": wo, "n_split": tile.get("n_split", 1)})
    seen, uniq = set(), []
    for t in out:
        key = (t["tile_n"], t["tile_h"], t["tile_w"])
        if key not in seen:
            seen.add(key)
            uniq.append(t)
    # prefer tiles near the planner's pixel count (keeps the search short)
    px0 = tile["tile_n"] * tile["tile_h"] * tile["tile_w"]
    rest = sorted(uniq[1:], key=lambda t: abs(t["tile_n"] * t["tile_h"] * t["tile_w"] - px0))
    sel = [uniq[0]] + rest[:limit - 1]
    # small maps (7^2, 14^2): a C_out split multiplies the CTAs (the DW stage is recomputed per
    # split, cheap at these sizes) when the tiles alone leave SMs idle or a ragged last wave
    if ho * wo <= 14 * 14 and cout >= 64:
        for t in list(sel[:3]):
            for ns in (2, 4):
                if cout // ns >= 16 and t.get("n_split", 1) == 1:
                    sel.append(dict(t, n_split=ns))
    return sel


def pwdw_tile_alternatives(tile, ho, wo, k, s, dtype, limit=10):
    """PWDW_R output tiles besides the planner's: the PW runs over the tile's halo, whose rows are
    the MMA rows (<= 512 for bf16/f16 -- 4 row blocks x 64 T columns x 2 TMEM buffers -- else 256);
    larger tiles recompute less halo, smaller ones give more tiles (measured, not modelled)."""
    rmax = 512 if dtype in ("bf16", "f16") else 256
    out = [dict(tile)]
    sizes = [4, 7, 8, 10, 12, 14, 16, 28]
    for th in sizes:
        for tw in sizes:
            th, tw = min(th, ho), min(tw, wo)
            th_in, tw_in = (th - 1) * s + k, (tw - 1) * s + k
            if th_in * tw_in > rmax or th * tw < 16:
                continue
            out.append({"tile_n": 1, "tile_h": th, "tile_w": tw, "n_split": tile.get("n_split", 1)})
    if k * k <= rmax:
        hw_in = ((ho - 1) * s + k) * ((wo - 1) * s + k)
        for nb in range(2, rmax // hw_in + 1):
            out.append({"tile_n": nb, "tile_h": ho, "tile_w": wo, "n_split": tile.get("n_split", 1)})
    seen, uniq = set(), []
    for t in out:
        key = (t["tile_n"], t["tile_h"], t["tile_w"])
        if key not in seen:
            seen.add(key)
            uniq.append(t)
    # largest outputs per halo row first (least recompute), then the rest
    def eff(t):
        r = t["tile_n"] * ((t["tile_h"] - 1) * s + k) * ((t["tile_w"] - 1) * s + k)
        return -t["tile_n"] * t["tile_h"] * t["tile_w"] / r
    rest = sorted(uniq[1:], key=eff)
    return [uniq[0]] + rest[:limit - 1]


def dw_tile_alternatives(tile, ho, wo, k, s, c, dtype):
    """LBL DW output tiles besides the planner's default: small tiles give more CTAs (latency
    hiding on small maps), large ones less halo; the measurement picks."""
    esize = {"f32": 4, "bf16": 2, "f16": 2, "s8": 1}[dtype]
    pb = min(128, c * esize)
    out, seen = [dict(tile)], {(tile["tile_h"], tile["tile_w"])}
    for th, tw in [(4, 7), (4, 8), (4, 16), (7, 7), (7, 14), (8, 8), (8, 14), (8, 16), (14, 14), (8, 32),
                   (16, 16), (16, 32), (28, 28)]:
        th, tw = min(th, ho), min(tw, wo)
        th_in, tw_in = (th - 1) * s + k, (tw - 1) * s + k
        if (th, tw) in seen or th_in > 256 or tw_in > 256 or th_in * tw_in * pb > 110 * 1024:
            continue
        seen.add((th, tw))
        out.append(dict(tile, tile_h=th, tile_w=tw))
    return out


def pwpw_candidates(model: dict, probe, dtype: str, batch: int):
    """FCM PWPW candidates: every producer -> consumer edge between two PW
    layers, with the §8(d)-style compulsory bytes (T never reaches HBM: 2 b |T| saved)."""
    esize = {"f32": 4, "bf16": 2, "f16": 2, "s8": 1}[dtype]
    kinds = {l["id"]: l for l in model["layers"]}
    out = []
    for a, b in model["edges"]:
        la, lb = kinds[a], kinds[b]
        if la["kind"] != "pw" or lb["kind"] != "pw" or la.get("extra_consumers", 0) or la.get("residual", 0):
            continue  # a shortcut reads a's output (it must reach HBM) / T would carry a residual
        m = batch * la["h"] * la["w"]
        cin, cmid, cout = la["c_in"], la["c_out"], lb["c_out"]
        dram = esize * (m * (cin + cout * (1 + lb.get("residual", 0))) + cin * cmid + cmid * cout)
        out.append({"op": "pwpw", "kind": "pwpw", "layers": [a, b], "tile": None, "dram_bytes": dram, "l2_bytes": dram,
                    "lbl_dram_bytes": dram + 2 * esize * m * cmid, "pred_us": 0.0,
                    "macs": m * (cin * cmid + cmid * cout)})
    return out


def refine(net: str, dtype: str, batch: int, device="cuda", reps=10, verbose=False, tile_search=True):
    plan = fcm.plan(model_json(net, dtype, batch))
    cands = plan["candidates"]
    # one Network instance whose "plan" is every candidate, so each has real buffers to run on
    all_entries = [dict(c) for c in cands["lbl"]] + [dict(c) for c in cands["fcm"]]
    probe = Network(net, dtype, batch, {"entries": []}, device=device)
    all_entries += pwpw_candidates(model_json(net, dtype, batch), probe, dtype, batch)
    order = probe.order
    meas, report = {}, []
    for c in all_entries:
        lids = c["layers"]
        l0 = probe.layers[lids[0]]
        cin = l0["c"] if l0["kind"] == "dw" else l0["c_in"]
        src = torch.zeros((batch, l0["h"], l0["w"], cin), dtype=probe.x.dtype, device=device)
        out = torch.empty(probe._out_shape(lids[-1]), dtype=probe.x.dtype, device=device)
        res = torch.zeros_like(out) if "residual_from" in probe.layers[lids[-1]] and dtype != "s8" else None
        tiles = [c.get("tile")]
        if tile_search and c["op"] == "dwpw" and c.get("tile"):
            d = probe.layers[lids[0]]
            kk, ss = d["k"], d["stride"]
            ho = (d["h"] + 2 * (kk // 2) - kk) // ss + 1
            wo = (d["w"] + 2 * (kk // 2) - kk) // ss + 1
            tiles = dwpw_tile_alternatives(c["tile"], ho, wo, kk, ss, probe.layers[lids[1]]["c_out"], dtype)
        elif tile_search and c["op"] == "pw" and c.get("tile") and dtype in ("bf16", "f16", "s8"):
            cout = probe.layers[lids[0]]["c_out"]
            tiles = [c["tile"]] + [dict(c["tile"], n_split=ns) for ns in (1, 2, 3, 4, 6, 8)
                                   if ns != c["tile"].get("n_split") and -(-cout // ns) >= 16 and -(-cout // ns) <= 256]
        elif tile_search and c["op"] == "pwdw_r" and c.get("tile") and dtype in ("bf16", "f16", "s8"):
            d = probe.layers[lids[1]]
            kk, ss = d["k"], d["stride"]
            ho = (d["h"] + 2 * (kk // 2) - kk) // ss + 1
            wo = (d["w"] + 2 * (kk // 2) - kk) // ss + 1
            tiles = pwdw_tile_alternatives(c["tile"], ho, wo, kk, ss, dtype)
        elif tile_search and c["op"] == "dw" and c.get("tile") and c["tile"].get("tile_w", 0) > 1:
            d = probe.layers[lids[0]]
            kk, ss = d["k"], d["stride"]
            ho = (d["h"] + 2 * (kk // 2) - kk) // ss + 1
            wo = (d["w"] + 2 * (kk // 2) - kk) // ss + 1
            tiles = dw_tile_alternatives(c["tile"], ho, wo, kk, ss, d["c"], dtype)
        best = None
        for t in tiles:
            ct = dict(c, tile=t) if t is not None else c
            f = probe._make_call(ct, src, out, res)
            try:
                us = _time(f, reps)
            except Exception as e:  # infeasible tile etc.: never chosen
                if verbose:
                    print("skip", lids, t, e)
                continue
            if best is None or us < best[0]:
                best = (us, t)
        if best is not None:
            report.append({"op": c["op"], "layers": lids, "tile": best[1], "us": round(best[0], 2)})
            meas[tuple(lids)] = best[0]
            if best[1] is not None:
                c["tile"] = best[1]
        del src, out, res
    lbl = {l: meas[(l,)] for l in order}
    fcm_cost = {k: v for k, v in meas.items() if len(k) == 2 and v < lbl[k[0]] + lbl[k[1]]}
    sel, total = chain_dp(order, lbl, fcm_cost)
    by_layers = {tuple(c["layers"]): c for c in all_entries}
    entries = []
    for s in sel:
        e = copy.deepcopy(by_layers[s])
        e["measured_us"] = meas[s]
        entries.append(e)
    out = dict(plan)
    out["entries"] = entries
    out["mode"] = "b200+measured"
    out["totals"] = dict(plan["totals"], measured_us=total, dram_bytes=sum(e["dram_bytes"] for e in entries),
                         fused_pairs=sum(1 for e in entries if len(e["layers"]) == 2))
    out.pop("candidates", None)
    out["measured_candidates"] = report
    return out


def verify_against_lbl(net: str, dtype: str, plan: dict, device="cuda", images: int = 4):
    """Run the chosen plan once on real (seeded) images and compare it with the all-LBL plan of
    the same stack: an FCM computes exactly PW(DW(X)) / DW(PW(X)) with T in the FM dtype (P:85,
    P:111), so int8 must match bit for bit and floats up to the R3b reassociation (rare
    1-ulp flips of T, far inside the 2e-2 / 1e-5 tolerances)."""
    lbl = {"entries": fcm.plan(model_json(net, dtype, images))["candidates"]["lbl"]}
    a = Network(net, dtype, images, {"entries": plan["entries"]}, device=device)
    a.run()
    b = Network(net, dtype, images, lbl, device=device)
    b.run()
    torch.cuda.synchronize()
    ya, yb = a.out.float(), b.out.float()
    same = bool(torch.equal(a.out, b.out))
    rel = float(((ya - yb).abs().max() / yb.abs().max().clamp_min(1e-30)).item())
    tol = 0.0 if dtype == "s8" else (1e-5 if dtype == "f32" else 2e-2)
    return {"images": images, "vs": "all-LBL plan on the GPU", "bit_identical": same,
            "max_abs_diff_over_max_abs": rel, "ok": bool(torch.isfinite(ya).all()) and (same or rel <= tol)}

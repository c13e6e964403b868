"""Time one FCM candidate with explicit tiles inside an otherwise layer-by-layer plan (development):
python tools/pwdw_probe.py --layers b1.0,b1.1 --op pwdw_r --tiles 14x8,7x14,8x7 [--trace]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_19331_b200 as fcm  # noqa: E402
from paper_2404_19331_b200.network import Network, model_json  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--net", default="mobilenet_v2")
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--layers", default="b1.0,b1.1")
ap.add_argument("--op", default="pwdw_r")
ap.add_argument("--tiles", default="")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
plan = fcm.plan(model_json(a.net, a.dtype, a.batch))
lids = a.layers.split(",")
cand = [c for c in plan["candidates"]["fcm"] if c["layers"] == lids and c["op"] == a.op][0]
lbl = {tuple(c["layers"]): c for c in plan["candidates"]["lbl"]}
for t in (a.tiles.split(",") if a.tiles else [""]):
    c = dict(cand)
    if t:
        parts = [int(v) for v in t.split("x")]
        c["tile"] = dict(c["tile"], tile_h=parts[0], tile_w=parts[1], tile_n=parts[2] if len(parts) > 2 else 1)
    ents, done = [], False
    for e in plan["entries"]:
        for l in e["layers"]:
            if l in lids:
                if not done:
                    ents.append(c)
                    done = True
            else:
                ents.append(lbl[(l,)])
    netw = Network(a.net, a.dtype, a.batch, dict(plan, entries=ents))
    i = next(j for j, inf in enumerate(netw.step_info) if inf["layers"] == lids)
    f = netw.steps[i]
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / a.reps
    print(f"{a.op} {a.layers} tile {c['tile']} {us:.2f} us  {netw.step_info[i]['dram_bytes'] / us / 1e3:.0f} GB/s")
    del netw

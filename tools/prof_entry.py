"""Run selected plan entries of a network (for ncu captures): python tools/prof_entry.py --entries 0,3"""
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
ap.add_argument("--entries", default="0")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--plan-file", default="")
ap.add_argument("--lbl", action="store_true", help="run the all layer-by-layer plan (one kernel per layer)")
ap.add_argument("--plan-out", default="", help="write the plan that runs (JSON)")
a = ap.parse_args()
import json  # noqa: E402
plan = json.load(open(a.plan_file)) if a.plan_file else fcm.plan(model_json(a.net, a.dtype, a.batch))
if a.lbl:
    full = fcm.plan(model_json(a.net, a.dtype, a.batch))
    lbl = {tuple(c["layers"]): c for c in full["candidates"]["lbl"]}
    plan = dict(plan, entries=[lbl[(l,)] for e in plan["entries"] for l in e["layers"]])
if a.plan_out:
    json.dump({k: v for k, v in plan.items() if k != "candidates"}, open(a.plan_out, "w"), indent=1)
netw = Network(a.net, a.dtype, a.batch, plan)
torch.cuda.synchronize()
ids = list(range(len(netw.steps))) if a.entries == "all" else [int(i) for i in a.entries.split(",")]
for i in ids:
    for _ in range(a.reps):
        netw.steps[i]()
    torch.cuda.synchronize()
    print(i, netw.step_info[i]["op"], netw.step_info[i]["layers"], netw.step_info[i]["tile"])

"""Time selected plan entries (CUDA events, L2-warm loop): python tools/time_entry.py --entries 22"""
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
ap.add_argument("--entries", default="22")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--plan-file", default="")
a = ap.parse_args()
import json  # noqa: E402
plan = json.load(open(a.plan_file)) if a.plan_file else fcm.plan(model_json(a.net, a.dtype, a.batch))
netw = Network(a.net, a.dtype, a.batch, plan)
ids = list(range(len(netw.steps))) if a.entries == "all" else [int(i) for i in a.entries.split(",")]
for i in ids:
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
    info = netw.step_info[i]
    us = e0.elapsed_time(e1) * 1e3 / a.reps
    print(f"{i:3d} {info['op']:7s} {','.join(info['layers']):12s} {us:9.2f}us {info['dram_bytes']/us/1e3:8.1f}GB/s tile {info['tile']}")

#!/usr/bin/env python
"""Benchmark: MobileNetV2 DW/PW stack (BASELINE configs[2]) on B200 through libfcm, images/sec.

One step = one pass of the whole FusePlanner-chosen stack (17 inverted residuals as FCMs DWPW /
PWDW_R + layer-by-layer PW, final PW 320->1280) over one batch of synthetic NHWC bf16 images,
replayed as one CUDA graph. `value` = images/sec over all ranks (weak scaling: 256 images per
GPU); timed with CUDA events on the launching stream, max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fcm|reference] [--net ...]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused DW+PW layer µs & HBM GB/s vs B200 peak; MobileNetV2 images/sec @1/2/4/8"
# BASELINE.json configs index of each network's stack (configs[0] is the single-layer parity case)
CONFIG_OF = {"single_dwpw": "configs[0]", "mobilenet_v1": "configs[1]", "mobilenet_v2": "configs[2]",
             "efficientnet_b0": "configs[3]", "cvt13": "configs[4]",
             "xception": "SURVEY 8(f) rank 2, 299x299", "ceit_leff": "SURVEY 8(f) rank 2",
             "cmt_irffn": "SURVEY 8(f) rank 2"}
DTYPE_NAME = {"bf16": "bf16", "f16": "f16", "s8": "s8", "f32": "f32"}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


# ------------------------------------------------------------------------------ clocks sampler
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx, self.proc, self.lines = gpu_index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------ energy
def energy_per_image(replay, images_per_replay, ms_per_replay, gpu_index, seconds=2.0):
    """Energy per inference, the analogue of the paper's energy experiment: NVML's
    cumulative board energy counter (mJ) read around >= `seconds` of back-to-back replays of the
    captured step. Board energy includes idle/static power, as a wall-socket meter would."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
        n = max(1, int(seconds * 1e3 / max(ms_per_replay, 1e-3)))
        torch.cuda.synchronize()
        t0, e0 = time.perf_counter(), pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        for _ in range(n):
            replay()
        torch.cuda.synchronize()
        t1, e1 = time.perf_counter(), pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        pynvml.nvmlShutdown()
        joules = (e1 - e0) / 1e3
        return {"j_per_image": round(joules / (n * images_per_replay), 6), "avg_power_w": round(joules / (t1 - t0), 1),
                "seconds": round(t1 - t0, 3), "images": n * images_per_replay,
                "method": "NVML total energy counter around back-to-back graph replays (board power)"}
    except Exception as e:  # reporting only; never fails the bench
        return {"error": str(e)[:200]}


# ------------------------------------------------------------------------------ helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def kernel_family(op, dtype=None, layer=None):
    """The kernel a plan entry launches. int8 stride-1 3x3 / 5x5 DW layers with a 16-byte pixel pitch
    on maps >= 14 x 14 (5x5: C <= 512) run the tensor-core DW (the dispatch rule of csrc/dw.cu)."""
    if op == "dw" and dtype == "s8" and layer is not None:
        k, s, c = layer["k"], layer["stride"], layer["c"]
        ho = (layer["h"] + 2 * (k // 2) - k) // s + 1
        wo = (layer["w"] + 2 * (k // 2) - k) // s + 1
        if s == 1 and k in (3, 5) and c % 16 == 0 and ho >= 14 and wo >= 14 and (k == 3 or c <= 512):
            return "dw_tc_i8_kernel"
    if dtype == "f32" and op == "pwdw_r":  # fp32 PWDW_R runs on FFMA (fp32 DWPW: the tensor-core kernel
        return "pwdw_simt_kernel"          # when its weight split fits shared memory)
    return {"dw": "dw_nhwc_kernel", "pw": "pw_tc_kernel", "dwpw": "dwpw_tc_kernel", "pwdw_r": "pwdw_tc_kernel",
            "pwpw": "pwpw_tc_kernel"}[op]


def per_entry_times(netw, reps=100):
    """Device time of every plan entry (one kernel each), SURVEY §8(d) protocol: before every
    timed launch a buffer of 2x the L2 size is written (outside the CUDA-event pair), so each launch
    starts L2-cold; `reps` launches per entry; median / p10 / p90 in microseconds."""
    st = torch.cuda.current_stream()
    l2 = torch.cuda.get_device_properties(st.device).L2_cache_size
    flush = torch.empty(2 * l2 // 4 + 1024, dtype=torch.float32, device=st.device)
    out = []
    for f in netw.steps:
        for _ in range(2):
            f()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        torch.cuda.synchronize()
        for a, b in ev:
            flush.zero_()
            a.record(st)
            f()
            b.record(st)
        torch.cuda.synchronize()
        us = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
        q = lambda p: us[min(len(us) - 1, int(p * (len(us) - 1) + 0.5))]
        out.append({"median": statistics.median(us), "p10": q(0.1), "p90": q(0.9), "reps": reps})
    del flush
    return out


def in_step_entry_times(netw, replays=20):
    """Device time of every plan entry INSIDE the step: the whole stack is captured once more with
    a pair of CUDA events (graph event-record nodes) around every launch, and this graph is
    replayed `replays` times; per entry the median over replays of its event pair, in
    microseconds. Inputs / L2 state are those of the real step (each layer reads what the
    previous one just wrote); the event nodes serialise neighbouring launches (no PDL overlap)."""
    st = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
          for _ in netw.steps]
    s = torch.cuda.Stream()
    s.wait_stream(st)
    with torch.cuda.stream(s):
        netw.run()
    st.wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for (a, b), f in zip(ev, netw.steps):
            a.record()
            f()
            b.record()
    samples = [[] for _ in netw.steps]
    for r in range(replays + 2):
        g.replay()
        torch.cuda.synchronize()
        if r >= 2:
            for i, (a, b) in enumerate(ev):
                samples[i].append(a.elapsed_time(b) * 1e3)
    return [statistics.median(x) for x in samples]


def host_cpu():
    """nproc and the lscpu model name of the host the oracle runs on."""
    model = None
    try:
        for ln in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if ln.lower().startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "model": model}


def cpu_baseline(net, dtype, seconds=15.0):
    """The oracle (oracle/network.py, numpy fp64 / exact int) as it stands on the host cores,
    on a bounded sample of the same workload: whole images through the whole stack, timed once
    with one BLAS thread and once with all cores (the oracle's only parallelism is numpy/BLAS)."""
    from oracle import network as on
    from threadpoolctl import threadpool_info, threadpool_limits
    prm = on.params(net, dtype)
    on.forward(net, dtype, 0, 1, prm=prm)  # warm-up (allocations, BLAS init)

    def run(limit, secs):
        with threadpool_limits(limits=limit):
            threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
            t0, n = time.perf_counter(), 0
            while time.perf_counter() - t0 < secs:
                on.forward(net, dtype, n, 1, prm=prm)
                n += 1
            return n / (time.perf_counter() - t0), n, threads
    v1, n1, _ = run(1, seconds / 3)
    va, na, threads = run(os.cpu_count(), 2 * seconds / 3)
    cpu = host_cpu()
    return {"value": va, "unit": "images/s", "cores": threads, "kind": "oracle",
            "single_thread": {"value": v1, "images": n1}, "host": cpu,
            "sample": f"{na} (all cores) + {n1} (1 thread) images x whole {net} DW/PW stack ({dtype}), one at a time, "
                      f"{seconds:.0f} s total"}


def cudnn_stack(net, dtype, batch, dev, steps=20, warmup=5, energy_gpu=None):
    """cuDNN's unfused DW + PW (PyTorch F.conv2d, channels_last, cudnn.benchmark) on the same layers
    and synthetic weights: BN scale folded into the weights, bias in the conv, activation in place
    (clamp / SiLU / GELU), the identity shortcuts as an add after the block's projection, stage /
    pooled maps fed like the FCM stack. Captured in a CUDA graph; device time per step via CUDA events."""
    import numpy as np
    import torch.nn.functional as F
    from synth.networks import NETWORKS, block_source, layer_ids, network_params
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}[dtype]
    torch.backends.cudnn.benchmark = True
    prm = network_params(0x5EED, net, dtype)
    blocks = NETWORKS[net]()
    layers = []
    for lid, bi, l in layer_ids(blocks):
        p = prm[lid]
        sc = torch.as_tensor(np.asarray(p["scale"]), dtype=torch.float64)
        if l["kind"] == "dw":
            w = torch.as_tensor(np.asarray(p["w"]), dtype=torch.float64).permute(2, 0, 1)[:, None] * sc[:, None, None, None]
        else:
            w = (torch.as_tensor(np.asarray(p["w"]), dtype=torch.float64).t() * sc[:, None])[:, :, None, None]
        layers.append((l["kind"], w.to(tdt).to(dev).contiguous(memory_format=torch.channels_last),
                       torch.as_tensor(np.asarray(p["bias"])).to(tdt).to(dev), l, lid, bi))
    maps = {}

    def stage_map(bi, l):
        cin = l["c"] if l["kind"] == "dw" else l["c_in"]
        key = (l["h"], l["w"], cin)
        if key not in maps:
            maps[key] = torch.randn(batch, cin, l["h"], l["w"], device=dev, dtype=tdt).contiguous(
                memory_format=torch.channels_last)
        return maps[key]

    def run():
        y = None
        inputs = {}
        for kind, w, b, l, lid, bi in layers:
            if y is None or (lid.endswith(".0") and block_source(net, blocks, bi)[0] == "stage"):
                y = stage_map(bi, l)
            inputs[lid] = y
            if kind == "dw":
                y = F.conv2d(y, w, b, stride=l["stride"], padding=l["k"] // 2, groups=l["c"])
            else:
                y = F.conv2d(y, w, b)
            if l["act"] == 2:
                y.clamp_(0, 6)
            elif l["act"] == 1:
                y.relu_()
            elif l["act"] == 3:
                y = F.silu(y, inplace=True)
            elif l["act"] == 4:
                y = F.gelu(y)
            if "residual_from" in l:
                y.add_(inputs[l["residual_from"]])
        return y
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    for _ in range(warmup):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    out = {"value": round(batch / (ms / 1e3), 1), "unit": "images/s", "ms_per_step": round(ms, 4),
           "kind": "torch F.conv2d (cuDNN), unfused DW + PW, folded BN, channels_last, CUDA graph"}
    if energy_gpu is not None:
        out["energy"] = energy_per_image(g.replay, batch, ms, energy_gpu)
    return out


def traffic_from_profiles(kernel, config_tag):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p))
        t = d.get(config_tag, {}).get(kernel)
        return None if t is None else round(t["traffic_bytes_per_launch"])
    except Exception:
        return None


# ------------------------------------------------------------------------------ reference arm
def run_reference(args, ws, rank):
    if rank != 0:
        return 0
    cb = None
    from oracle import network as on
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    prm = on.params(args.net, args.dtype)
    per_step = max(1, args.ref_images)
    for i in range(args.warmup):
        on.forward(args.net, args.dtype, i, 1, prm=prm)
    t0 = time.perf_counter()
    for k in range(args.steps):
        on.forward(args.net, args.dtype, k * per_step, per_step, prm=prm)
    dt = time.perf_counter() - t0
    v = args.steps * per_step / dt
    cb = {"value": v, "unit": "images/s", "cores": cores, "kind": "oracle",
          "sample": f"{per_step} image(s) per step x {args.steps} steps, whole {args.net} stack ({args.dtype})"}
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "images/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic", "config": {"workload": f"{args.net} DW/PW stack "
                                                        f"({CONFIG_OF.get(args.net, 'not a BASELINE config')}), "
                                                        f"{args.batch} img/GPU",
                                            "net": args.net, "global_batch": ws * args.batch,
                                            "images_per_step": per_step,
                                            "sample": "the oracle processes a bounded sample of the batch per step"},
            "cpu_baseline": cb, "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


class _Eager2:
    """Stands in for a CUDA graph when launching eagerly (ncu launch lists)."""

    def __init__(self, net):
        self.net = net

    def replay(self):
        self.net.run()


# ------------------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="fcm", choices=["fcm", "reference"])
    ap.add_argument("--net", default="mobilenet_v2")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--batch", type=int, default=256, help="images per GPU")
    ap.add_argument("--mode", default="b200", choices=["b200", "paper"])
    ap.add_argument("--plan", default="measured", choices=["measured", "model", "all-dwpw"],
                    help="measured: refine the planner's choice with timed candidates (autotune.refine); "
                         "all-dwpw: every DW layer fused with its PW consumer (configs[1]'s 'FCM DWPW on "
                         "every block'), whether or not it is faster")
    ap.add_argument("--plan-out", default="", help="write the executed plan (JSON) here")
    ap.add_argument("--ref-images", type=int, default=1, help="reference arm: images per step")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cudnn", action="store_true", help="skip the cuDNN unfused DW+PW baseline")
    ap.add_argument("--layers-out", default="", help="write the per-entry table (JSON) here")
    ap.add_argument("--no-graph", action="store_true", help="launch eagerly (for ncu launch lists)")
    ap.add_argument("--no-energy", action="store_true", help="skip the NVML energy-per-image measurement")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    ws, rank, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `python bench.py --gpus N` without torchrun: spawn the N ranks ourselves
        from paper_2404_19331_b200.replicas import relaunch_under_torchrun
        relaunch_under_torchrun(args.gpus, [os.path.abspath(__file__)] + sys.argv[1:])
    if ws != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}: launch one rank per GPU")
    if args.impl == "reference":
        return run_reference(args, ws, rank)

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    import paper_2404_19331_b200 as fcm
    from paper_2404_19331_b200.network import Network, model_json
    from paper_2404_19331_b200 import replicas

    n0, _ = replicas.shard(args.batch, ws, rank)
    plan_verify = None
    if args.plan == "measured" and args.mode == "b200":
        # rank 0 measures; every rank executes the same plan (so the shards are bit-identical to
        # a one-GPU run of the same plan and the post-timing verification is meaningful)
        plan = None
        if rank == 0:
            from paper_2404_19331_b200.autotune import refine, verify_against_lbl
            plan = refine(args.net, args.dtype, args.batch, device=dev)
            plan_verify = verify_against_lbl(args.net, args.dtype, plan, device=dev)
        plan = replicas.broadcast_plan(plan, ws)
    elif args.plan == "all-dwpw":
        plan = fcm.plan(model_json(args.net, args.dtype, args.batch, args.mode))
        cands = plan["candidates"]
        lbl = {c["layers"][0]: c for c in cands["lbl"]}
        dwpw = {c["layers"][0]: c for c in cands["fcm"] if c["op"] == "dwpw"}
        order = [c["layers"][0] for c in cands["lbl"]]
        ents, i = [], 0
        while i < len(order):
            if order[i] in dwpw and i + 1 < len(order) and dwpw[order[i]]["layers"][1] == order[i + 1]:
                ents.append(dwpw[order[i]])
                i += 2
            else:
                ents.append(lbl[order[i]])
                i += 1
        plan = dict(plan, entries=ents, mode="all-dwpw",
                    totals=dict(plan["totals"], fused_pairs=sum(len(e["layers"]) == 2 for e in ents),
                                dram_bytes=sum(e["dram_bytes"] for e in ents)))
        plan.pop("candidates", None)
        if rank == 0:
            from paper_2404_19331_b200.autotune import verify_against_lbl
            plan_verify = verify_against_lbl(args.net, args.dtype, plan, device=dev)
    else:
        plan = fcm.plan(model_json(args.net, args.dtype, args.batch, args.mode))
    if args.plan_out and rank == 0:
        with open(args.plan_out, "w") as f:
            json.dump(plan, f, indent=1)
    netw = Network(args.net, args.dtype, args.batch, plan, device=dev, n0=n0)
    if args.no_graph:
        netw.run()
        torch.cuda.synchronize()

        graph = _Eager2(netw)
    else:
        graph = netw.capture()
    launches_per_step = len(netw.steps)
    st = torch.cuda.current_stream()

    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()

    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.15)

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    # ---------------- device-resident timed region
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        graph.replay()
    e1.record(st)
    torch.cuda.synchronize()
    barrier()
    t_ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    energy = None
    if not args.no_energy and not args.no_graph:
        energy = energy_per_image(graph.replay, args.batch, t_ms / args.steps, local)

    # ---------------- end-to-end through the public API with host buffers
    # Every step copies its batch host->device (pinned) and its output device->host inside the
    # timed region. Two input/output buffer sets (two captured instances of the same plan) let the
    # H2D copy of step k+1 and the D2H copy of step k-1 run on copy streams while step k computes.
    x_host = netw.x.cpu().pin_memory()
    y_host = [torch.empty(netw.out.shape, dtype=netw.out.dtype).pin_memory() for _ in range(2)]
    nets = [netw, Network(args.net, args.dtype, args.batch, plan, device=dev, n0=n0)]
    graphs = [graph, (nets[1].capture() if not args.no_graph else _Eager2(nets[1]))]
    cin, cout = torch.cuda.Stream(), torch.cuda.Stream()
    in_ready = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    out_read = [torch.cuda.Event() for _ in range(2)]

    def e2e_steps_run(n):
        for k in range(n):
            i = k & 1
            with torch.cuda.stream(cin):
                if k >= 2:
                    cin.wait_event(done[i])          # step k-2 no longer reads nets[i].x
                nets[i].x.copy_(x_host, non_blocking=True)
                in_ready[i].record(cin)
            st.wait_event(in_ready[i])
            if k >= 2:
                st.wait_event(out_read[i])           # step k-2's output already copied out
            graphs[i].replay()
            done[i].record(st)
            with torch.cuda.stream(cout):
                cout.wait_event(done[i])
                y_host[i].copy_(nets[i].out, non_blocking=True)
                out_read[i].record(cout)
        st.wait_stream(cin)
        st.wait_stream(cout)

    e2e_steps_run(4)
    torch.cuda.synchronize()
    e2e_steps = max(10, args.steps // 4)
    barrier()
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(st)
    e2e_steps_run(e2e_steps)
    a1.record(st)
    torch.cuda.synchronize()
    barrier()
    t_e2e = a0.elapsed_time(a1)
    e2e_same = bool(torch.equal(y_host[0], y_host[1]))  # both buffer sets ran the same batch and plan

    # ---------------- per-entry (per-kernel) device times
    entry_stats = per_entry_times(netw)          # isolated launches, L2-cold, 100 reps each
    times_us = in_step_entry_times(netw)         # the same launches inside the step (roofline)

    t_ms, t_e2e = replicas.max_over_ranks([t_ms, t_e2e], dev, ws)
    if ws > 1:
        # verification only (after timing): per-image checksums over NCCL; rank 0 recomputes the
        # first images of every shard with its own Network instance
        def run_probe(p0, n):
            probe = Network(args.net, args.dtype, n, plan, device=dev, n0=p0)
            probe.run()
            return probe.out
        verify = replicas.verify_shards(netw.out, args.batch, ws, rank, run_probe)

    pk = peaks()
    hbm_peak = float(pk.get("hbm_gbs", 6650.0))
    fam = {}
    rows = []
    # binding roof: per launch max(t_HBM, t_DW on the FFMA pipe, t_PW on the
    # tensor cores); DW peak = SMs x 128 fp32 MAC/clk x max SM clock (the FFMA/FFMA2 rate,
    # tools/microbench/fma_rates.cu); PW peak = measured dense bf16 (f16 same, int8 2x, tf32 1/2)
    sm_hz = float(pk.get("sm_max_mhz", 1965.0)) * 1e6
    dw_mac_s = 148 * 128 * sm_hz
    tc_mac_s = float(pk.get("bf16_tflops", 1598.4)) * 1e12 / 2 * {"s8": 2.0, "f32": 0.5}.get(args.dtype, 1.0)
    for info, us, es in zip(netw.step_info, times_us, entry_stats):
        k = kernel_family(info["op"], args.dtype, netw.layers[info["layers"][0]])
        f = fam.setdefault(k, {"us": 0.0, "bytes": 0, "n": 0, "bind_us": 0.0, "t": {"hbm": 0.0, "dw_alu": 0.0, "pw_tc": 0.0}})
        f["us"] += us
        f["bytes"] += info["dram_bytes"]
        f["n"] += 1
        t = {"hbm": info["dram_bytes"] / (hbm_peak * 1e3),
             "dw_alu": info.get("dw_macs", 0) / dw_mac_s * 1e6,
             "pw_tc": (info.get("pw_macs", 0) + info.get("redundant_macs", 0) + info.get("macs", 0)) / tc_mac_s * 1e6}
        f["bind_us"] += max(t.values())
        for kk in t:
            f["t"][kk] += t[kk]
        rows.append({"op": info["op"], "layers": info["layers"], "tile": info.get("tile"), "us": round(us, 3),
                     "cold_us": round(es["median"], 3), "cold_p10": round(es["p10"], 3), "cold_p90": round(es["p90"], 3),
                     "dram_bytes": info["dram_bytes"], "l2_bytes": info["l2_bytes"],
                     "lbl_dram_bytes": info["lbl_dram_bytes"],
                     "gbs": round(info["dram_bytes"] / us / 1e3, 1), "frac_hbm": round(info["dram_bytes"] / us / 1e3 / hbm_peak, 3),
                     "pred_us": round(info["pred_us"], 3)})
    dom = max(fam, key=lambda k: fam[k]["us"])
    d = fam[dom]
    achieved = d["bytes"] / d["us"] / 1e3  # GB/s
    sum_us = sum(times_us)

    if rank == 0:
        ms_per_step = t_ms / args.steps
        value = ws * args.batch * args.steps / (t_ms / 1e3)
        in_bytes = netw.x.numel() * netw.x.element_size()
        out_bytes = netw.out.numel() * netw.out.element_size()
        config_tag = f"{args.net}/{args.dtype}/b{args.batch}"
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "images/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (seeded splitmix64 inputs/weights, random-init)",
            "config": {"workload": f"{args.net} DW/PW stack ({CONFIG_OF.get(args.net, 'not a BASELINE config')}), "
                                   f"{args.batch} img/GPU",
                       "net": args.net, "global_batch": ws * args.batch, "plan_mode": plan["mode"],
                       "fused_pairs": plan["totals"]["fused_pairs"], "kernels_per_step": launches_per_step,
                       "parallelism": f"batch-sharded x{ws} (replicas, no collective on the hot path)",
                       "l2": "inputs larger than L2 (205 MB input + 2.8 GB compulsory traffic per step)",
                       "planned_dram_bytes_per_step": plan["totals"]["dram_bytes"],
                       "lbl_dram_bytes_per_step": plan["totals"]["lbl_dram_bytes"]},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": hbm_peak,
                         "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                         "traffic": traffic_from_profiles(dom, config_tag),
                         "share_of_step": round(d["us"] / sum_us, 3), "launches_per_step": d["n"],
                         "timing": "CUDA events around every launch inside the captured step (median of 20 replays); "
                                   "isolated L2-cold medians (100 launches, 2x L2 flushed before each) in the layers file",
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" + (" (fallback)" if pk.get("_fallback") else "")},
            "binding_roof": {"kernel": dom, "t_us": {kk: round(v, 2) for kk, v in d["t"].items()},
                             "bound": max(d["t"], key=d["t"].get), "measured_us": round(d["us"], 2),
                             "frac": round(d["bind_us"] / d["us"], 4),
                             "peaks": {"hbm_gbs": hbm_peak, "dw_fp32_tmac_s": round(dw_mac_s / 1e12, 1),
                                       "pw_tc_tmac_s": round(tc_mac_s / 1e12, 1)}},
            "stack_hbm": {"achieved_gbs": round(plan["totals"]["dram_bytes"] / (ms_per_step * 1e-3) / 1e9, 1),
                          "frac": round(plan["totals"]["dram_bytes"] / (ms_per_step * 1e-3) / 1e9 / hbm_peak, 4)},
            "e2e": {"value": round(ws * args.batch * e2e_steps / (t_e2e / 1e3), 1), "unit": "images/s",
                    "h2d_bytes_per_step": in_bytes, "d2h_bytes_per_step": out_bytes,
                    "overlap": "H2D (pinned) and D2H on copy streams overlap the previous / next step's "
                               "kernels; 2 buffer sets", "outputs_identical": e2e_same},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk,
        }
        if energy is not None:
            line["energy"] = energy
        if ws > 1:
            line["verify"] = verify
        if plan_verify is not None:
            line["plan_verify"] = plan_verify
        if not args.no_cudnn and args.dtype in ("bf16", "f16", "f32"):
            try:
                cb = cudnn_stack(args.net, args.dtype, args.batch, dev,
                                 energy_gpu=None if (args.no_energy or energy is None) else local)
                if cb:
                    cb["fcm_speedup"] = round(line["value"] / ws / cb["value"], 3)
                    ce, fe = cb.get("energy", {}), line.get("energy", {})
                    if "j_per_image" in ce and "j_per_image" in fe and fe["j_per_image"] > 0:
                        cb["fcm_energy_ratio"] = round(fe["j_per_image"] / ce["j_per_image"], 3)
                    line["cudnn_baseline"] = cb
            except Exception as e:  # baseline only; never fails the bench
                line["cudnn_baseline"] = {"error": str(e)[:200]}
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args.net, args.dtype, args.cpu_seconds)
        if args.layers_out:
            with open(args.layers_out, "w") as f:
                json.dump({"config": config_tag, "rows": rows, "families": fam, "plan_totals": plan["totals"]}, f,
                          indent=1)
        for r in rows:
            print(f"{r['op']:7s} {','.join(r['layers']):12s} {r['us']:9.2f}us cold {r['cold_us']:.1f} [{r['cold_p10']:.1f},{r['cold_p90']:.1f}] {r['gbs']:8.1f}GB/s "
                  f"frac {r['frac_hbm']:.3f} pred {r['pred_us']:8.2f}us tile {r['tile']}", file=sys.stderr)
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

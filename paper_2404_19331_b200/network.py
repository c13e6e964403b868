"""DW/PW network stacks executed from a FusePlanner plan (CNNs assembled from FCM and
layer-by-layer kernels chosen by the planner).

A `Network` owns device weights (PW weights packed offline), epilogue vectors and
activation buffers, and a list of steps -- each one call into libfcm (fcm_dw / fcm_pw /
fcm_dwpw / fcm_pwdw_r), i.e. exactly one kernel launch. The whole stack can be captured into
one CUDA graph and replayed. Inputs and parameters are synthetic (synth/), keyed by global
image index so that batch shards are exact slices of one global batch.
"""
from __future__ import annotations

import dataclasses

import numpy as np
import torch

import synth
from synth.networks import NETWORKS, block_source, layer_ids, network_params
import paper_2404_19331_b200 as fcm

TORCH_DT = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16, "s8": torch.int8}
ESIZE = {"f32": 4, "bf16": 2, "f16": 2, "s8": 1}


def model_json(net: str, dtype: str, batch: int, mode: str = "b200", shortcuts: bool = True) -> dict:
    """Planner input for a named network: the layer list plus producer->consumer edges.
    shortcuts=False drops the residual adds (the paper's DW/PW-only model, SURVEY App. A byte pins);
    int8 stacks never carry them (no int8 residual epilogue, reading R1b)."""
    shortcuts = shortcuts and dtype != "s8"
    blocks = NETWORKS[net]()
    ids = layer_ids(blocks)
    out = []
    for lid, _, l in ids:
        if l["kind"] == "dw":
            k = l["k"]
            out.append({"id": lid, "kind": "dw", "h": l["h"], "w": l["w"], "c": l["c"], "k": k,
                        "stride": l["stride"], "pads": [k // 2] * 4})
        else:
            out.append({"id": lid, "kind": "pw", "h": l["h"], "w": l["w"], "c_in": l["c_in"],
                        "c_out": l["c_out"]})
            if shortcuts and "residual_from" in l:
                out[-1]["residual"] = 1  # the epilogue reads one output-shaped shortcut tensor
    edges = []
    for i in range(1, len(ids)):
        (a, ba, _), (c, bc, _) = ids[i - 1], ids[i]
        if ba == bc or block_source(net, blocks, bc)[0] == "chain":
            edges.append([a, c])
    if shortcuts:
        # the shortcut re-reads the producer's output: a second consumer, so that output is never an
        # FCM intermediate (single-consumer rule, reading R20)
        by_id = {l["id"]: l for l in out}
        for lid, _, l in ids:
            src = l.get("residual_from")
            for a, c in edges if src else ():
                if c == src:
                    by_id[a]["extra_consumers"] = by_id[a].get("extra_consumers", 0) + 1
    return {"dtype": dtype, "batch": batch, "mode": mode, "layers": out, "edges": edges}


def stored(a: np.ndarray, dtype: str) -> torch.Tensor:
    """Cast generated values to the storage dtype (CPU tensor)."""
    if dtype == "s8":
        return torch.from_numpy(np.asarray(a, dtype=np.int64)).to(torch.int8)
    return torch.from_numpy(np.asarray(a, dtype=np.float64)).to(TORCH_DT[dtype])


def input_images(net: str, dtype: str, role: str, n0: int, n: int, h: int, w: int, c: int,
                 seed: int = synth.SEED) -> torch.Tensor:
    kind = "int8" if dtype == "s8" else "float"
    return stored(synth.activations(seed, role, n0, n, h, w, c, kind), dtype)


class Network:
    def __init__(self, net: str, dtype: str, batch: int, plan: dict, device="cuda", seed=synth.SEED, n0: int = 0):
        self.net, self.dtype, self.batch, self.plan, self.dev, self.seed, self.n0 = \
            net, dtype, batch, plan, device, seed, n0
        self.blocks = NETWORKS[net]()
        ids = layer_ids(self.blocks)
        self.layers = {lid: dict(l, block=bi) for lid, bi, l in ids}
        self.order = [lid for lid, _, _ in ids]
        self.params = {}
        self._make_params()
        first = self.layers[self.order[0]]
        c0 = first["c"] if first["kind"] == "dw" else first["c_in"]
        self.x = input_images(net, dtype, f"{net}/input", n0, batch, first["h"], first["w"], c0, seed).to(device)
        self.steps, self.step_info = [], []
        self._build_steps()

    def _make_params(self):
        dev = self.dev
        for lid, p in network_params(self.seed, self.net, self.dtype).items():
            l = self.layers[lid]
            if self.dtype == "s8":
                i32 = lambda a: torch.as_tensor(np.asarray(a), dtype=torch.int32, device=dev)
                ep = fcm.Epilogue(act=l["act"], bias_q=i32(p["bias_q"]), mult_q=i32(p["mult_q"]),
                                  shift_q=i32(p["shift_q"]), zp_in=0, zp_out=0, qmin=p["qmin"], qmax=p["qmax"])
            else:
                f32 = lambda a: torch.as_tensor(np.asarray(a), dtype=torch.float32, device=dev)
                ep = fcm.Epilogue(act=l["act"], scale=f32(p["scale"]), bias=f32(p["bias"]))
            w = stored(p["w"], self.dtype).to(dev)
            if l["kind"] == "pw":
                w = fcm.pack_pw(w)
            self.params[lid] = (w, ep)

    def _out_shape(self, lid):
        l = self.layers[lid]
        if l["kind"] == "dw":
            ho = (l["h"] + 2 * (l["k"] // 2) - l["k"]) // l["stride"] + 1
            wo = (l["w"] + 2 * (l["k"] // 2) - l["k"]) // l["stride"] + 1
            return (self.batch, ho, wo, l["c"])
        return (self.batch, l["h"], l["w"], l["c_out"])

    def _entries(self):
        """Plan entries as launched: a paper-mode FCM entry the fused kernels cannot run
        ("executable": false -- k outside {3, 5} or no kernel tile) runs as its LBL layers."""
        for e in self.plan["entries"]:
            if e.get("executable", True) or len(e["layers"]) == 1:
                yield e
            else:
                for lid in e["layers"]:
                    yield {"op": self.layers[lid]["kind"], "kind": self.layers[lid]["kind"], "layers": [lid]}

    def _build_steps(self):
        cur = self.x
        stage_in = {}
        entry_in = {}  # first layer of an entry -> its input tensor (shortcut sources)
        self.outputs, self.inputs, self.entries, self.residuals = [], [], [], []
        for e in self._entries():
            lids = e["layers"]
            l0 = self.layers[lids[0]]
            bi = l0["block"]
            first_of_block = lids[0] == f"b{bi}.0"
            src = cur
            if first_of_block:
                kind, role = block_source(self.net, self.blocks, bi)
                if kind == "stage":
                    c = l0["c"] if l0["kind"] == "dw" else l0["c_in"]
                    if role not in stage_in:
                        stage_in[role] = self.x if bi == 0 else input_images(
                            self.net, self.dtype, role, self.n0, self.batch, l0["h"], l0["w"], c, self.seed).to(self.dev)
                    src = stage_in[role]
            out = torch.empty(self._out_shape(lids[-1]), dtype=TORCH_DT[self.dtype], device=self.dev)
            entry_in[lids[0]] = src
            rf = self.layers[lids[-1]].get("residual_from") if self.dtype != "s8" else None
            if rf is not None and rf not in entry_in:
                raise ValueError(f"plan hides the shortcut source {rf} of {lids[-1]} inside a fused entry")
            res = entry_in[rf] if rf is not None else None
            self.steps.append(self._make_call(e, src, out, res))
            self.residuals.append(res)
            self.step_info.append(dict(e, in_shape=tuple(src.shape), out_shape=tuple(out.shape)))
            cur = out
            self.outputs.append(out)
            self.inputs.append(src)
            self.entries.append(e)
        self.out = cur

    def _make_call(self, e, src, out, res=None):
        """One libfcm call for plan entry e; `res` = the shortcut tensor added by the entry's output
        epilogue, or None."""
        op, lids, tile = e["op"], e["layers"], e.get("tile")
        withres = (lambda ep: ep) if res is None else (lambda ep: dataclasses.replace(ep, residual=res))
        if op == "dw":
            l = self.layers[lids[0]]
            w, ep = self.params[lids[0]]
            return lambda: fcm.dw(src, w, l["stride"], None, ep, out=out, tile=tile)
        if op == "pw":
            w, ep = self.params[lids[0]]
            ep = withres(ep)
            return lambda: fcm.pw(src, w, ep, out=out, tile=tile)
        if op == "dwpw":
            l = self.layers[lids[0]]
            (wd, ed), (wp, ep) = self.params[lids[0]], self.params[lids[1]]
            ep = withres(ep)
            return lambda: fcm.dwpw(src, wd, l["stride"], None, ed, wp, ep, out=out, tile=tile)
        if op == "pwpw":
            (w1, e1), (w2, e2) = self.params[lids[0]], self.params[lids[1]]
            e2 = withres(e2)
            return lambda: fcm.pwpw(src, w1, e1, w2, e2, out=out)
        if op == "pwdw_r":
            l = self.layers[lids[1]]
            (wp, ep), (wd, ed) = self.params[lids[0]], self.params[lids[1]]
            return lambda: fcm.pwdw_r(src, wp, ep, wd, l["stride"], None, ed, out=out, tile=tile)
        raise ValueError(op)

    def run(self):
        for f in self.steps:
            f()
        return self.out

    def capture(self):
        """Capture the whole stack into one CUDA graph (launch-bound small layers)."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.run()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.run()
        self.graph = g
        return g

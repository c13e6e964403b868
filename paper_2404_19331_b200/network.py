"""DW/PW network stacks executed from a FusePlanner plan (CNNs assembled from FCM and
layer-by-layer kernels chosen by the planner).

A `Network` owns device weights (PW weights packed offline), epilogue vectors and
activation buffers, and a list of steps -- each one call into libfcm (fcm_dw / fcm_pw /
fcm_dwpw / fcm_pwdw_r). The whole stack can be captured into one CUDA graph and replayed.
Inputs are synthetic (synth/), keyed by global image index so batch shards are exact slices.
"""
from __future__ import annotations

import numpy as np
import torch

import synth
from synth.networks import NETWORKS
import paper_2404_19331_b200 as fcm

TORCH_DT = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16, "s8": torch.int8}
ESIZE = {"f32": 4, "bf16": 2, "f16": 2, "s8": 1}


def layer_list(blocks):
    """Flatten blocks into a chain of layers with ids '<block>.<i>' and resolved pads/out dims."""
    layers = []
    for bi, b in enumerate(blocks):
        for li, l in enumerate(b):
            d = dict(l)
            d["id"] = f"b{bi}.{li}"
            d["block"] = bi
            layers.append(d)
    return layers


def model_json(net: str, dtype: str, batch: int, mode: str = "b200") -> dict:
    """Planner input for a named network (edges: each block is a chain; blocks chain too,
    except CvT whose Q/K/V projections each start from the block input)."""
    blocks = NETWORKS[net]()
    layers = layer_list(blocks)
    out = []
    for l in layers:
        if l["kind"] == "dw":
            k = l["k"]
            out.append({"id": l["id"], "kind": "dw", "h": l["h"], "w": l["w"], "c": l["c"], "k": k,
                        "stride": l["stride"], "pads": [k // 2] * 4})
        else:
            out.append({"id": l["id"], "kind": "pw", "h": l["h"], "w": l["w"], "c_in": l["c_in"],
                        "c_out": l["c_out"]})
    edges = []
    for i in range(1, len(layers)):
        a, b = layers[i - 1], layers[i]
        if a["block"] == b["block"] or net != "cvt13":
            edges.append([a["id"], b["id"]])
    return {"dtype": dtype, "batch": batch, "mode": mode, "layers": out, "edges": edges}


class Network:
    def __init__(self, net: str, dtype: str, batch: int, plan: dict, device="cuda", seed=synth.SEED, n0: int = 0):
        self.net, self.dtype, self.batch, self.plan, self.dev = net, dtype, batch, plan, device
        blocks = NETWORKS[net]()
        self.layers = {l["id"]: l for l in layer_list(blocks)}
        self.order = [l["id"] for l in layer_list(blocks)]
        self.seed = seed
        self.params = {}
        self._make_params()
        first = self.layers[self.order[0]]
        c0 = first["c"] if first["kind"] == "dw" else first["c_in"]
        self.in_shape = (batch, first["h"], first["w"], c0)
        kind = "int8" if dtype == "s8" else "float"
        x = synth.activations(seed, f"{net}/input", n0, batch, first["h"], first["w"], c0, kind)
        self.x = (torch.from_numpy(x.astype(np.int64)).to(torch.int8) if dtype == "s8"
                  else torch.from_numpy(x).to(TORCH_DT[dtype])).to(device)
        self.steps = []
        self.step_info = []
        self._build_steps()

    # ------------------------------------------------------------------ parameters
    def _make_params(self):
        s, dt, dev = self.seed, self.dtype, self.dev
        sigma = 73.9
        for lid in self.order:
            l = self.layers[lid]
            name = f"{self.net}/{lid}"
            if dt == "s8":
                if l["kind"] == "dw":
                    p = synth.int8_dw_params(s, name, l["k"], l["c"], l["act"], sigma)
                else:
                    p = synth.int8_pw_params(s, name, l["c_in"], l["c_out"], l["act"], sigma)
                sigma = 32.0
                i32 = lambda a: torch.as_tensor(np.asarray(a), dtype=torch.int32, device=dev)
                ep = fcm.Epilogue(act=l["act"], bias_q=i32(p["bias_q"]), mult_q=i32(p["mult_q"]),
                                  shift_q=i32(p["shift_q"]), zp_in=0, zp_out=0, qmin=p["qmin"], qmax=p["qmax"])
                w = torch.as_tensor(p["w"], dtype=torch.int8).to(dev)
            else:
                if l["kind"] == "dw":
                    p = synth.float_dw_params(s, name, l["k"], l["c"], l["act"])
                else:
                    p = synth.float_pw_params(s, name, l["c_in"], l["c_out"], l["act"])
                f32 = lambda a: torch.as_tensor(np.asarray(a), dtype=torch.float32, device=dev)
                ep = fcm.Epilogue(act=l["act"], scale=f32(p["scale"]), bias=f32(p["bias"]))
                w = torch.from_numpy(p["w"]).to(TORCH_DT[dt]).to(dev)
            if l["kind"] == "pw":
                w = fcm.pack_pw(w)
            self.params[lid] = (w, ep, p)

    # ------------------------------------------------------------------ steps
    def _out_shape(self, lid):
        l = self.layers[lid]
        if l["kind"] == "dw":
            ho = (l["h"] + 2 * (l["k"] // 2) - l["k"]) // l["stride"] + 1
            wo = (l["w"] + 2 * (l["k"] // 2) - l["k"]) // l["stride"] + 1
            return (self.batch, ho, wo, l["c"])
        return (self.batch, l["h"], l["w"], l["c_out"])

    def _build_steps(self):
        cur = self.x
        stage_in = {}  # CvT: every Q/K/V projection of a stage reads that stage's token map
        for e in self.plan["entries"]:
            lids = e["layers"]
            l0 = self.layers[lids[0]]
            first_of_block = lids[0] == [i for i in self.order if self.layers[i]["block"] == l0["block"]][0]
            if self.net == "cvt13" and first_of_block:
                key = (l0["h"], l0["c"])
                if key not in stage_in:
                    stage_in[key] = self.x if tuple(self.x.shape[1:]) == (l0["h"], l0["w"], l0["c"]) \
                        else self._fresh_in(l0)
                src = stage_in[key]
            else:
                src = cur
            out = torch.empty(self._out_shape(lids[-1]), dtype=TORCH_DT[self.dtype], device=self.dev)
            self.steps.append(self._make_call(e, src, out))
            self.step_info.append(dict(e, in_shape=tuple(src.shape), out_shape=tuple(out.shape)))
            cur = out
        self.out = cur

    def _fresh_in(self, l0):
        c = l0["c"] if l0["kind"] == "dw" else l0["c_in"]
        kind = "int8" if self.dtype == "s8" else "float"
        x = synth.activations(self.seed, f"{self.net}/in{l0['id']}", 0, self.batch, l0["h"], l0["w"], c, kind)
        return (torch.from_numpy(x.astype(np.int64)).to(torch.int8) if self.dtype == "s8"
                else torch.from_numpy(x).to(TORCH_DT[self.dtype])).to(self.dev)

    def _make_call(self, e, src, out):
        op = e["op"]
        lids = e["layers"]
        tile = e.get("tile")
        if op == "dw":
            l = self.layers[lids[0]]
            w, ep, _ = self.params[lids[0]]
            return lambda: fcm.dw(src, w, l["stride"], None, ep, out=out, tile=tile)
        if op == "pw":
            w, ep, _ = self.params[lids[0]]
            return lambda: fcm.pw(src, w, ep, out=out)
        if op == "dwpw":
            l = self.layers[lids[0]]
            wd, ed, _ = self.params[lids[0]]
            wp, ep, _ = self.params[lids[1]]
            return lambda: fcm.dwpw(src, wd, l["stride"], None, ed, wp, ep, out=out, tile=tile)
        if op == "pwdw_r":
            l = self.layers[lids[1]]
            wp, ep, _ = self.params[lids[0]]
            wd, ed, _ = self.params[lids[1]]
            return lambda: fcm.pwdw_r(src, wp, ep, wd, l["stride"], None, ed, out=out, tile=tile)
        raise ValueError(op)

    def run(self):
        for f in self.steps:
            f()
        return self.out

    def capture(self):
        """Capture the whole stack into a CUDA graph (launch-bound small layers)."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.run()  # warm (sets smem attributes, caches device props)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.run()
        self.graph = g
        return g

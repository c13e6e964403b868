"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no convolution, no epilogue, no
rounding of results). It only produces random numbers and the layer shapes of the
paper's workloads:

* a counter-based generator (splitmix64 over (seed, role, global element index)),
  so that any slice of a tensor -- e.g. one rank's batch shard -- is regenerated
  bit-identically without generating the rest;
* value recipes per dtype:
  float  X ~ U(-1,1); W_dw ~ U(-1,1)*sqrt(3/k^2); W_pw ~ U(-1,1)*sqrt(3/C_in);
         scale ~ U(0.5,1.5); bias ~ U(-0.1,0.1)
  int8   X ~ U{-128..127}; W ~ U{-127..127}; bias_q ~ U{-4096..4096};
         per-channel fixed-point multiplier (M in [2^30, 2^31), shift) chosen so the
         requantised output has sigma ~ 32 LSB;
* the DW/PW layer tables of the BASELINE networks (synth.networks).

Values are returned as numpy arrays (float64 for float recipes, int64 for int8
recipes). Conversion to a storage dtype is done by the caller with a plain cast
(torch .to(dtype)); both the oracle and the CUDA path then read the SAME stored bits.
"""
from __future__ import annotations

import math

import numpy as np

SEED = 0x5EED
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def fnv1a64(s: str) -> int:
    h = 0xCBF29CE484222325
    for b in s.encode():
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def _key(seed: int, role: str) -> np.uint64:
    with np.errstate(over="ignore"):
        return _mix(np.array([(seed ^ fnv1a64(role)) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0]


def bits(seed: int, role: str, n: int, offset: int = 0) -> np.ndarray:
    """n uint64 words: element i is splitmix64 output number (offset+i) of stream (seed, role)."""
    idx = np.arange(offset, offset + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = _key(seed, role) + (idx + np.uint64(1)) * _GOLDEN
        return _mix(z)


def uniform(seed: int, role: str, shape, lo: float, hi: float, offset: int = 0) -> np.ndarray:
    n = int(np.prod(shape)) if len(shape) else 1
    u = (bits(seed, role, n, offset) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return (lo + (hi - lo) * u).reshape(shape)


def randint(seed: int, role: str, shape, lo: int, hi: int, offset: int = 0) -> np.ndarray:
    """Integers uniform in [lo, hi] (inclusive)."""
    n = int(np.prod(shape)) if len(shape) else 1
    span = np.uint64(hi - lo + 1)
    return (lo + (bits(seed, role, n, offset) % span).astype(np.int64)).reshape(shape)


# ----------------------------------------------------------------------------------
# activations: NHWC, keyed by global image index so batch shards regenerate exactly
# ----------------------------------------------------------------------------------
def activations(seed: int, role: str, n0: int, n: int, h: int, w: int, c: int, kind: str) -> np.ndarray:
    """Images [n0, n0+n) of an NHWC activation tensor. kind: 'float' | 'int8'."""
    per = h * w * c
    if kind == "int8":
        return randint(seed, role, (n, h, w, c), -128, 127, offset=n0 * per)
    return uniform(seed, role, (n, h, w, c), -1.0, 1.0, offset=n0 * per)


# ----------------------------------------------------------------------------------
# layer parameters
# ----------------------------------------------------------------------------------
ACT_NONE, ACT_RELU, ACT_RELU6, ACT_SILU, ACT_GELU = 0, 1, 2, 3, 4
INT8_RELU6_QMAX = 96  # synthetic output scale: real 6.0 <-> 96 LSB


def float_dw_params(seed: int, name: str, k: int, c: int, act: int) -> dict:
    a = math.sqrt(3.0 / (k * k))
    return dict(w=uniform(seed, name + "/w_dw", (k, k, c), -a, a),
                scale=uniform(seed, name + "/scale", (c,), 0.5, 1.5),
                bias=uniform(seed, name + "/bias", (c,), -0.1, 0.1), act=act)


def float_pw_params(seed: int, name: str, c_in: int, c_out: int, act: int) -> dict:
    a = math.sqrt(3.0 / c_in)
    return dict(w=uniform(seed, name + "/w_pw", (c_in, c_out), -a, a),
                scale=uniform(seed, name + "/scale", (c_out,), 0.5, 1.5),
                bias=uniform(seed, name + "/bias", (c_out,), -0.1, 0.1), act=act)


def _fixed_point(seed: int, role: str, eff: float, c: int):
    """Per-channel (M, shift) with M in [2^30, 2^31) and M/2^shift ~ eff*U(0.8,1.25)."""
    s = eff * uniform(seed, role, (c,), 0.8, 1.25)
    e = np.floor(np.log2(s)).astype(np.int64)
    sh = 30 - e
    m = np.floor(s * np.exp2(sh.astype(np.float64))).astype(np.int64)
    m = np.clip(m, 1 << 30, (1 << 31) - 1)
    return m, sh


def int8_quant(seed: int, name: str, c_out: int, fan_in: int, act: int, sigma_in: float = 73.9,
               zp_in: int = 0, zp_out: int = 0) -> dict:
    eff = 32.0 / (math.sqrt(fan_in) * sigma_in * 73.3)
    m, sh = _fixed_point(seed, name + "/mult", eff, c_out)
    if act == ACT_NONE:
        qmin, qmax = -128, 127
    elif act == ACT_RELU:
        qmin, qmax = zp_out, 127
    else:
        qmin, qmax = zp_out, min(127, zp_out + INT8_RELU6_QMAX)
    return dict(bias_q=randint(seed, name + "/bias_q", (c_out,), -4096, 4096), mult_q=m, shift_q=sh,
                zp_in=zp_in, zp_out=zp_out, qmin=qmin, qmax=qmax, act=act)


def int8_dw_params(seed: int, name: str, k: int, c: int, act: int, sigma_in: float = 73.9) -> dict:
    p = int8_quant(seed, name, c, k * k, act, sigma_in)
    p["w"] = randint(seed, name + "/w_dw", (k, k, c), -127, 127)
    return p


def int8_pw_params(seed: int, name: str, c_in: int, c_out: int, act: int, sigma_in: float = 73.9) -> dict:
    p = int8_quant(seed, name, c_out, c_in, act, sigma_in)
    p["w"] = randint(seed, name + "/w_pw", (c_in, c_out), -127, 127)
    return p

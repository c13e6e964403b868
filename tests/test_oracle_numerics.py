"""Pins for oracle/numerics.py against independent library routines and hand values."""
import json
import os

import numpy as np
import torch

from oracle.numerics import requant, round_to

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rand_doubles(n, seed=1):
    rng = np.random.default_rng(seed)
    mant = rng.uniform(-1, 1, n)
    exp = rng.integers(-30, 20, n)
    return np.ldexp(mant, exp)


def test_f16_matches_numpy_cast():
    x = _rand_doubles(200000)
    # include ties at fp16 precision, subnormals and overflow
    ties = (np.arange(-2000, 2000) + 0.5) * 2.0 ** -10
    sub = (np.arange(-300, 300) + 0.5) * 2.0 ** -24
    big = np.array([65504.0, 65519.99, 65520.0, 70000.0, -65520.0])
    x = np.concatenate([x, ties, sub, big])
    ours = round_to(x, "f16")
    ref = x.astype(np.float16).astype(np.float64)
    assert np.array_equal(ours, ref)


def test_f32_matches_numpy_cast():
    x = np.concatenate([_rand_doubles(200000, 2), np.ldexp(np.arange(1, 999) + 0.5, -170)])
    assert np.array_equal(round_to(x, "f32"), x.astype(np.float32).astype(np.float64))


def test_bf16_matches_torch_cast_of_float32():
    rng = np.random.default_rng(3)
    raw = rng.integers(0, 2 ** 32, 400000, dtype=np.uint64).astype(np.uint32)
    # force exact ties (lower 16 bits 0x8000) for a quarter of them
    raw[::4] = (raw[::4] & np.uint32(0xFFFF0000)) | np.uint32(0x8000)
    f = raw.view(np.float32)
    f = f[np.isfinite(f)]
    ref = torch.from_numpy(f.copy()).to(torch.bfloat16).to(torch.float64).numpy()
    ours = round_to(f.astype(np.float64), "bf16")
    assert np.array_equal(ours, ref)


def test_requant_hand_values():
    g = json.load(open(os.path.join(GOLD, "worked_vectors.json")))
    for acc, m, sh, want in g["requant_hand"]:
        assert int(requant(acc, m, sh)) == want
    # round half toward +inf (arithmetic shift): ties go up for both signs
    assert int(requant(12, 1 << 30, 33)) == 2   # 1.5 -> 2
    assert int(requant(-12, 1 << 30, 33)) == -1  # -1.5 -> -1


def test_requant_matches_python_bigint():
    rng = np.random.default_rng(5)
    acc = rng.integers(-(1 << 30), 1 << 30, 5000)
    m = rng.integers(1 << 30, 1 << 31, 5000)
    sh = rng.integers(1, 62, 5000)
    got = requant(acc, m, sh)
    for a, mm, s, g in zip(acc.tolist(), m.tolist(), sh.tolist(), got.tolist()):
        # floor((a*m)/2^s + 1/2) written with Python big ints
        assert g == (2 * a * mm + (1 << s)) // (1 << (s + 1))

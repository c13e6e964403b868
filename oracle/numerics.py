"""Storage-format rounding and int8 requantisation (TEST INFRASTRUCTURE -- see oracle/__init__).

round_to(x, fmt)
    Round float64 values to the nearest value of the storage format, ties to even (IEEE
    754 roundTiesToEven), with gradual underflow and overflow to +-inf. The paper only
    evaluates FP32 and INT8; bf16/fp16 are BASELINE additions (north_star
    tolerance list), read as RNE storage (reading R11).
    Pinned by tests/test_oracle_numerics.py against numpy's float16/float32 casts and
    torch's float32->bfloat16 cast (independent library routines).

requant(acc, mult, shift)
    The paper never states its quantisation scheme (reading R1). We use the
    fixed-point requantiser  (acc * M + 2^(shift-1)) >> shift  (arithmetic shift, i.e.
    round half toward +inf), M in [2^30, 2^31), shift in [1, 62]. Pinned by hand values.
"""
from __future__ import annotations

import numpy as np

# (significand bits incl. the implicit one, emin, emax)
FORMATS = {"bf16": (8, -126, 127), "f16": (11, -14, 15), "f32": (24, -126, 127)}


def round_rne(x: np.ndarray, p: int, emin: int, emax: int) -> np.ndarray:
    """Round to a binary format with p significand bits and normal exponent range [emin, emax]."""
    x = np.asarray(x, dtype=np.float64)
    _, e = np.frexp(x)                      # x = m * 2^e, 0.5 <= |m| < 1
    lead = np.maximum(e - 1, emin)          # exponent of the leading bit (clamped: subnormals)
    ulp = np.exp2((lead - (p - 1)).astype(np.float64))
    r = np.rint(x / ulp) * ulp              # np.rint = round half to even
    maxfin = (2.0 - 2.0 ** (1 - p)) * 2.0 ** emax
    r = np.where(np.abs(r) > maxfin, np.copysign(np.inf, x), r)
    return np.where(x == 0, x, r)


def round_to(x: np.ndarray, fmt: str) -> np.ndarray:
    if fmt == "f64":
        return np.asarray(x, dtype=np.float64)
    p, emin, emax = FORMATS[fmt]
    return round_rne(x, p, emin, emax)


def requant(acc, mult, shift):
    """(acc*M + 2^(shift-1)) >> shift, exact (numpy int64; |acc| < 2^31, M < 2^31)."""
    acc = np.asarray(acc, dtype=np.int64)
    mult = np.asarray(mult, dtype=np.int64)
    shift = np.asarray(shift, dtype=np.int64)
    assert np.all(np.abs(acc) < (1 << 31)), "accumulator out of the exactness range"
    return (acc * mult + (np.int64(1) << (shift - 1))) >> shift

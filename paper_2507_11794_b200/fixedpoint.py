"""Host side of the i32 fixed-point codec (gpu/fixedpoint.py:25-66).

The device encodes with ``rint(f32(x) * f32(scale))`` saturating at
+-FIXED_SATURATION inside the kernels (cs_common.cuh ``encode_fixed``).  The
host needs the same codec for ``Engine.inject_response`` (engine.py:354-358)
and for decoding ``read_forces_raw`` / ``read_accumulator_raw``.
"""

from __future__ import annotations

import numpy as np

FIXED_SATURATION = 2147483520  # largest f32 below 2^31 (fixedpoint.py:25)


def encode_values(values, scale: int, float32: bool = True) -> np.ndarray:
    """i32(round-half-even(value * scale)), saturating (fixedpoint.py:28-41)."""
    values = np.asarray(values)
    if float32:
        product = values.astype(np.float32) * np.float32(scale)
        rounded = np.rint(product).astype(np.float64)
    else:
        rounded = np.rint(np.asarray(values, dtype=np.float64) * float(scale))
    with np.errstate(invalid="ignore"):
        clipped = np.clip(rounded, -FIXED_SATURATION, FIXED_SATURATION)
        out = clipped.astype(np.int64).astype(np.int32)
    return out


def decode_values(raw, scale: int, float32: bool = True) -> np.ndarray:
    """Exact decode to float64, optionally rounded once to f32 (fixedpoint.py:44-47)."""
    exact = np.asarray(raw, dtype=np.float64) / float(scale)
    return exact.astype(np.float32) if float32 else exact

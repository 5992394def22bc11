"""Deterministic synthetic inputs shared by the golden generator, tests and bench.

All values are bf16-representable so that the float64 CPU reference and the
bf16 GPU path see *identical* numbers.  Generation is pure
numpy (PCG64 streams are stable across machines and numpy versions), so the
golden fixtures produced in the build container match what the GPU box
regenerates.
"""

from __future__ import annotations

import numpy as np


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even); returns float32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return rounded.astype(np.uint32).view(np.float32)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """uint16 bit patterns of bf16-representable float32 values."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    return (x.view(np.uint32) >> 16).astype(np.uint16)


def bf16_from_bits(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint32) << 16).view(np.float32)


def randn_bf16(shape, seed: int) -> np.ndarray:
    """N(0,1) float32 draws rounded to bf16 (float32 container)."""
    rng = np.random.default_rng(seed)
    return bf16_round(rng.standard_normal(size=shape, dtype=np.float32))


def tie_heavy_bf16(shape, seed: int, levels: int = 3) -> np.ndarray:
    """Small-integer weights: many equal scores and gains (exercise every tie-break)."""
    rng = np.random.default_rng(seed)
    return rng.integers(-levels, levels + 1, size=shape).astype(np.float32)


def random_sigma_o(m: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).permutation(m).astype(np.int64)


def permute_survivors(survivors, seed: int):
    """sigma_i^t = ascending survivors of tile t permuted by a per-tile stream (seed + t)."""
    out = []
    for t, s in enumerate(survivors):
        s = np.asarray(s, dtype=np.int64)
        out.append(s[np.random.default_rng(seed + t).permutation(s.size)])
    return out

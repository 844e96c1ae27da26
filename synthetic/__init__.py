"""Seeded synthetic input generator shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no mixing, no weights, no update):
only the counter-based generator both sides use to build identical inputs.
The CUDA library carries its own implementation of the same generator
(``bf_fill_uniform`` in csrc/generate.cu); tests check the two bit for bit.

Generator (SURVEY.md §8(d) "Synthetic input generator"):
    v     = splitmix64(seed * 2**32 + idx)
    value = ((v >> 40) - 2**23) * 2**-23 * scale      uniform in [-1, 1) * scale,
exactly representable in fp32 for scale = 2**-k.

Seed recipe:
    x0 of agent r            : 1000 + r
    gradient of agent r, k   : 2000 + 7919*k + r   (scale 2**-7)
    A_i (least squares)      : 3000 + r            (scale 1/sqrt(m))
    x_natural                : 4000
    noise of agent r         : 5000 + r            (scale 0.01)
"""
from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)

SEED_X0 = 1000
SEED_G = 2000
SEED_A = 3000
SEED_XNAT = 4000
SEED_NOISE = 5000


def splitmix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser of (z + golden gamma); uint64 in, uint64 out (wrapping)."""
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z += _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform(seed: int, count: int, scale: float = 1.0, offset: int = 0) -> np.ndarray:
    """fp32 array of `count` values for elements offset..offset+count-1 of stream `seed`."""
    idx = np.arange(offset, offset + count, dtype=np.uint64)
    base = np.uint64((int(seed) << 32) & 0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        v = splitmix64(idx + base)
    q = (v >> np.uint64(40)).astype(np.int64) - (1 << 23)
    out = q.astype(np.float64) * (2.0 ** -23)
    if scale != 1.0:
        out = out * float(np.float32(scale))
    return out.astype(np.float32)


def grad_seed(step: int, rank: int) -> int:
    return SEED_G + 7919 * int(step) + int(rank)


def agents_x0(n: int, count: int) -> np.ndarray:
    """Stacked X^0, shape (n, count) fp32, row r from seed 1000 + r."""
    return np.stack([uniform(SEED_X0 + r, count) for r in range(n)])


def agents_grad(n: int, count: int, step: int) -> np.ndarray:
    """Stacked synthetic gradients for `step`, shape (n, count) fp32, scale 2**-7."""
    return np.stack([uniform(grad_seed(step, r), count, scale=2.0 ** -7) for r in range(n)])


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    """Decode bfloat16 bit patterns (uint16) to fp32 values (exact)."""
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32)

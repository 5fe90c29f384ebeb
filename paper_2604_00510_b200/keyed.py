"""Vectorised keyed splitmix64 folds for host-side problem tables.

The reference draws every random quantity from ``mix(*keys)`` — a splitmix64
fold over an integer key tuple (rng.py:15-27) — one Python call per draw.
Building a 65,536-request problem table that way costs seconds, so the host
side here folds whole key MATRICES at once with numpy uint64 arithmetic
(wraparound multiply is exactly the reference's ``& 2**64-1``).  The device
replays the same fold per expansion in csrc/engine.cu.
"""

from __future__ import annotations

import math

import numpy as np

_U = np.uint64
_SEED0 = _U(0x8E12F5A34C29D96B)
_GOLD = _U(0x9E3779B97F4A7C15)
_M1 = _U(0xBF58476D1CE4E5B9)
_M2 = _U(0x94D049BB133111EB)


def _sm(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + _GOLD
        x = (x ^ (x >> _U(30))) * _M1
        x = (x ^ (x >> _U(27))) * _M2
    return x ^ (x >> _U(31))


def fold_rows(keys) -> np.ndarray:
    """mix() of every row of an (n, k) integer key matrix → (n,) uint64."""
    k = np.asarray(keys, dtype=object)
    if k.ndim == 1:
        k = k[None, :]
    mat = np.array([[int(v) & 0xFFFFFFFFFFFFFFFF for v in row] for row in k], dtype=np.uint64) \
        if k.dtype == object else k.astype(np.uint64)
    h = np.full(mat.shape[0], _SEED0, dtype=np.uint64)
    for c in range(mat.shape[1]):
        h = _sm(h ^ mat[:, c])
    return h


def fold_columns(*cols) -> np.ndarray:
    """mix() over broadcast key columns (scalars or uint64 arrays)."""
    arrs = np.broadcast_arrays(*[np.asarray(c, dtype=np.uint64) for c in cols]) if cols else []
    h = np.full(arrs[0].shape if cols else (), _SEED0, dtype=np.uint64)
    for a in arrs:
        h = _sm(h ^ a)
    return h


def mix(*keys: int) -> int:
    """Scalar mix() (rng.py:22-27)."""
    return int(fold_columns(*[_U(int(k) & 0xFFFFFFFFFFFFFFFF) for k in keys]))


def to_unit(h) -> np.ndarray:
    """(h >> 11) * 2**-53 (rng.py:30-32); exact in float64."""
    return (np.asarray(h, dtype=np.uint64) >> _U(11)).astype(np.float64) * (2.0 ** -53)


def exponential_draw(rate: float, *keys: int) -> float:
    """-log1p(-u)/rate (rng.py:47-52), libm log1p like the reference."""
    if rate <= 0.0:
        raise ValueError("rate must be positive")
    return -math.log1p(-float(to_unit(mix(*keys)))) / rate


def keyed_permutation(items: list, seed: int, tag: int) -> list:
    """Fisher-Yates driven by mix(seed, tag, i) % (i+1) (rng.py:55-61);
    the draws are folded in one vectorised pass, the swaps are sequential."""
    out = list(items)
    n = len(out)
    if n < 2:
        return out
    idx = np.arange(n - 1, 0, -1, dtype=np.uint64)
    draws = fold_columns(_U(seed & 0xFFFFFFFFFFFFFFFF), _U(tag), idx)
    for i, d in zip(range(n - 1, 0, -1), draws.tolist()):
        j = d % (i + 1)
        out[i], out[j] = out[j], out[i]
    return out

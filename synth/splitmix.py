"""Counter-based SplitMix64 (Steele, Lea & Flood 2014), vectorised over numpy uint64.

This module holds NO arithmetic of the method (arXiv 1605.02043); it only draws
seeded pseudo-random numbers. Both the oracle tests and the CUDA path consume its
outputs, so it lives in its own package (`synth/`), imported by neither
`oracle/` nor `paper_1605_02043_b200/`.

    x_i   = seed + (i + 1) * 0x9E3779B97F4A7C15          (mod 2^64)
    z     = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9
    z     = (z ^ (z >> 27)) * 0x94D049BB133111EB
    out_i = z ^ (z >> 31)
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, counter: np.ndarray) -> np.ndarray:
    """Return SplitMix64 output number `counter` (0-based) of the stream `seed`."""
    c = np.asarray(counter).astype(np.uint64, copy=False)
    with np.errstate(over="ignore"):
        x = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (c + np.uint64(1)) * _GOLDEN
        z = (x ^ (x >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def uniform01(seed: int, counter: np.ndarray) -> np.ndarray:
    """Uniform doubles in [0, 1): top 53 bits of the SplitMix64 output."""
    return (splitmix64(seed, counter) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def uniform(seed: int, counter: np.ndarray, lo: float, hi: float) -> np.ndarray:
    return lo + (hi - lo) * uniform01(seed, counter)


def random_permutation(seed: int, n: int) -> np.ndarray:
    """A seeded permutation of range(n): position j holds the old id that gets new id j.

    Sort by 64-bit SplitMix64 keys (ties broken by id, stable), so it is O(n log n)
    in numpy and reproducible on any machine."""
    keys = splitmix64(seed, np.arange(n, dtype=np.uint64))
    try:
        import torch
        if torch.cuda.is_available() and n > (1 << 22):
            # same order as numpy's stable argsort of the unsigned keys: flip the sign bit so
            # that signed int64 order is unsigned order; stable, so equal keys keep id order
            k = (keys ^ np.uint64(1 << 63)).view(np.int64)
            return torch.sort(torch.from_numpy(k).cuda(), stable=True)[1].cpu().numpy().astype(np.int64)
    except ImportError:
        pass
    return np.argsort(keys, kind="stable").astype(np.int64)

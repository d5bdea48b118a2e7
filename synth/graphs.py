"""Small fixture graphs and seeded random graphs (inputs only; no method arithmetic).

Vertex ids are 0-based; the list index of an edge is its task id."""
from __future__ import annotations

import numpy as np

from .splitmix import splitmix64


def _e(pairs):
    return np.asarray(pairs, dtype=np.int32).reshape(-1, 2)


def fig_mot():
    """PAPER.md P:53-74 (fig:mot), reading Z1 of SURVEY §8(c): particles 1..6 -> 0..5,
    e1=(1,2) e2=(1,3) e3=(5,6) e4=(1,4) e5=(4,5) e6=(4,6)."""
    return 6, _e([(0, 1), (0, 2), (4, 5), (0, 3), (3, 4), (3, 5)])


def fig_mot_alt():
    """Second topology consistent with fig:mot's counts: particle 1 adjacent to all
    others plus (5,6): e1=(1,2) e2=(1,3) e3=(5,6) e4=(1,4) e5=(1,5) e6=(1,6)."""
    return 6, _e([(0, 1), (0, 2), (4, 5), (0, 3), (0, 4), (0, 5)])


def two_triangle():
    """"0 1/1 2/3 4/0 2/4 5/3 5"."""
    return 6, _e([(0, 1), (1, 2), (3, 4), (0, 2), (4, 5), (3, 5)])


def path_graph(m: int):
    return m + 1, _e([(i, i + 1) for i in range(m)])


def cycle_graph(m: int, offset: int = 0):
    return m, _e([(offset + i, offset + (i + 1) % m) for i in range(m)])


def random_multigraph(seed: int, m: int, n: int):
    """m edges with endpoints uniform in [0, n); self-loops and parallel edges kept."""
    r = splitmix64(seed, np.arange(2 * m, dtype=np.uint64))
    ends = (r % np.uint64(n)).astype(np.int32)
    return n, ends.reshape(m, 2)


def int_vector(seed: int, n: int, lo: int, hi: int) -> np.ndarray:
    """Integer-valued float32 vector, entries uniform in {lo..hi} (exact in fp32 sums)."""
    r = splitmix64(seed, np.arange(n, dtype=np.uint64))
    return (lo + (r % np.uint64(hi - lo + 1)).astype(np.int64)).astype(np.float32)

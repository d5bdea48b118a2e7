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


def rmat(scale: int, edge_factor: int = 8, seed: int = 1607, a=0.57, b=0.19, c=0.19, chunk: int = 1 << 22):
    """R-MAT edge list (Chakrabarti et al.): n = 2^scale vertices, m = edge_factor * n edges,
    quadrant probabilities (a, b, c, d = 1 - a - b - c) per level; duplicates and self-loops
    kept ('avg degree 16' read as 2m/n = 16, i.e. edge_factor 8).

    Level l of edge e uses 16 bits of SplitMix64 draw (e * ceil(scale/4) + l // 4)."""
    n = 1 << scale
    m = edge_factor * n
    per = (scale + 3) // 4
    ta, tab, tabc = int(a * 65536), int((a + b) * 65536), int((a + b + c) * 65536)
    out = np.empty((m, 2), dtype=np.int32)
    for e0 in range(0, m, chunk):
        e1 = min(m, e0 + chunk)
        cnt = e1 - e0
        base = (np.arange(e0, e1, dtype=np.uint64) * np.uint64(per))
        u = np.zeros(cnt, np.int64)
        v = np.zeros(cnt, np.int64)
        for w in range(per):
            r = splitmix64(seed, base + np.uint64(w))
            for j in range(4):
                lvl = 4 * w + j
                if lvl >= scale:
                    break
                q = ((r >> np.uint64(16 * j)) & np.uint64(0xFFFF)).astype(np.int64)
                bit = np.int64(1) << np.int64(scale - 1 - lvl)
                down = (q >= tab)                  # quadrants c, d: row bit set
                right = ((q >= ta) & (q < tab)) | (q >= tabc)   # quadrants b, d: column bit set
                u += bit * down
                v += bit * right
        out[e0:e1, 0] = u
        out[e0:e1, 1] = v
    return n, out


def stencil2d_spmv(g: int, chunk_rows: int = 1 << 22):
    """2D 5-point Laplacian on a g x g grid as the bipartite data-affinity graph of SpMV
    (P:859-861): vertices 0..N-1 are x_j (columns), N..2N-1 are y_i (rows), one edge
    (j, N + i) per nonzero A[i, j] in row-major (CUSP) order; values 4 / -1.
    Row i's nonzeros sit in columns i - g, i - 1, i, i + 1, i + g (ascending), so row-major
    order needs no sort; built in chunks of rows (g = 10,000: 499,960,000 nonzeros)."""
    N = g * g
    offs = np.array([-g, -1, 0, 1, g], np.int64)
    vals5 = np.array([-1.0, -1.0, 4.0, -1.0, -1.0], np.float32)
    ok_r = np.array([[-1, 0], [0, -1], [0, 0], [0, 1], [1, 0]], np.int64)
    parts_e, parts_v = [], []
    for i0 in range(0, N, chunk_rows):
        i = np.arange(i0, min(N, i0 + chunk_rows), dtype=np.int64)
        r, c = i // g, i % g
        ok = np.ones((i.size, 5), bool)
        for q, (dr, dc) in enumerate(ok_r):
            ok[:, q] = (r + dr >= 0) & (r + dr < g) & (c + dc >= 0) & (c + dc < g)
        cols = (i[:, None] + offs[None, :])[ok]
        rows = np.broadcast_to(i[:, None], (i.size, 5))[ok]
        parts_e.append(np.stack([cols, N + rows], axis=1).astype(np.int32))
        parts_v.append(np.broadcast_to(vals5[None, :], (i.size, 5))[ok])
    return 2 * N, np.concatenate(parts_e), np.concatenate(parts_v)

"""Brute-force helpers for the oracle pins (test infrastructure).

Independent of oracle/: loads are recounted with Python sets straight from Eq. (1)
(PAPER.md P:259-275), and balanced maps are enumerated exhaustively."""
from __future__ import annotations

from collections import defaultdict


def loads_and_cut(edges, part):
    """(L, C) by direct recount: L = sum_p |V_p|; C = sum_v (p_v - 1) over touched v."""
    V = defaultdict(set)
    clusters_of = defaultdict(set)
    for (u, v), p in zip(edges.tolist() if hasattr(edges, "tolist") else edges, list(part)):
        V[p].update((u, v))
        clusters_of[u].add(p)
        clusters_of[v].add(p)
    L = sum(len(s) for s in V.values())
    C = sum(len(s) - 1 for s in clusters_of.values())
    return L, C


def t_cut(t_ptr, t_adj, t_w, part):
    """Weighted cut of the task graph T under `part` (each undirected edge once)."""
    cut = 0
    for t in range(len(t_ptr) - 1):
        for q in range(t_ptr[t], t_ptr[t + 1]):
            nb = int(t_adj[q])
            if nb > t and part[t] != part[nb]:
                cut += int(t_w[q])
    return cut


def balanced_maps(sizes):
    """All assignments of tasks 0..m-1 to clusters with exact sizes, canonicalised
    (SPEC S:445): among clusters of equal target size, a cluster may only be opened
    after every lower-indexed cluster of that size is non-empty."""
    m = sum(sizes)
    k = len(sizes)
    fill = [0] * k
    cur = [0] * m

    def rec(t):
        if t == m:
            yield list(cur)
            return
        for b in range(k):
            if fill[b] >= sizes[b]:
                continue
            if fill[b] == 0 and any(sizes[c] == sizes[b] and fill[c] == 0 for c in range(b)):
                continue
            fill[b] += 1
            cur[t] = b
            yield from rec(t + 1)
            fill[b] -= 1

    yield from rec(0)


def optimum(edges, sizes, T=None):
    """(C*, T-cut*) over all balanced maps; T-cut* only if T = (t_ptr, t_adj, t_w)."""
    best_c, best_t = None, None
    for x in balanced_maps(sizes):
        _, c = loads_and_cut(edges, x)
        best_c = c if best_c is None else min(best_c, c)
        if T is not None:
            tc = t_cut(*T, x)
            best_t = tc if best_t is None else min(best_t, tc)
    return best_c, best_t

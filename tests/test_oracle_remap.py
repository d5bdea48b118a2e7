"""Pins for the oracle's remap (O6: task reorganisation + cpack)
and multi-GPU halo sets (O7)."""
import numpy as np
import pytest

import oracle as O
import synth as S
from conftest import golden


def cpack_sequential(edges, n, part, k, key=None):
    """cpack as the sequential first-touch walk of SPEC S:381 (a different formulation
    from the oracle's key sort): clusters ascending, tasks ascending (by (key, id) with a
    key, reading Z22), endpoints (u, v); each object gets the next free position on first
    touch; untouched appended by id."""
    new = -np.ones(n, np.int64)
    nxt = 0
    block_begin = []
    for p in range(k):
        block_begin.append(nxt)
        tasks = np.nonzero(part == p)[0]
        if key is not None:
            tasks = sorted(tasks.tolist(), key=lambda e: (key[e], e))
        for e in tasks:
            for v in edges[e]:
                if new[v] < 0:
                    new[v] = nxt
                    nxt += 1
    block_begin.append(nxt)
    for v in range(n):
        if new[v] < 0:
            new[v] = nxt
            nxt += 1
    return new, np.array(block_begin)


def check_layout(edges, n, part, k, lay, key=None):
    m = edges.shape[0]
    # 1. edge order by (part, id), or (part, key, id) (reading Z22)
    order = np.lexsort((np.arange(m), part)) if key is None else np.lexsort((np.arange(m), key, part))
    assert np.array_equal(lay.edge_perm, order)
    assert np.array_equal(lay.part_edge_begin, np.concatenate([[0], np.cumsum(np.bincount(part, minlength=k))]))
    # 2-4. cpack vs the sequential walk
    new, bb = cpack_sequential(edges, n, part, k, key)
    assert np.array_equal(lay.vertex_perm, new)
    assert np.array_equal(lay.part_vertex_begin, bb)
    assert sorted(lay.vertex_perm.tolist()) == list(range(n))            # bijection
    pvb = lay.part_vertex_begin
    assert pvb[0] == 0 and np.all(np.diff(pvb) >= 0)
    assert pvb[k] == len(set(edges.ravel().tolist()))                     # = touched
    # 5-7. halos and slots
    r = O.cost(edges, n, part, k)
    assert lay.halo_begin[k] == r.cut_cost == lay.halo_ids.size           # sum |H_p| = C
    total_loads = 0
    for p in range(k):
        H = lay.halo_ids[lay.halo_begin[p]:lay.halo_begin[p + 1]]
        assert np.all(np.diff(H) > 0) and np.all(H < pvb[p])
        nown = pvb[p + 1] - pvb[p]
        total_loads += nown + H.size
        for i in range(lay.part_edge_begin[p], lay.part_edge_begin[p + 1]):
            for s in range(2):
                sl = int(lay.slots[i, s])
                v_new = pvb[p] + sl if sl < nown else H[sl - nown]
                assert v_new == lay.vertex_perm[edges[lay.edge_perm[i], s]]   # slots dereference
    assert total_loads == r.load_count                                    # remap keeps L


def test_two_triangle_block_begin():
    g = golden("two_triangle.json")
    e = np.array(g["edges"], np.int32)
    part = np.array(g["optimal_partition"], np.int32)
    lay = O.remap(e, 6, part, 2)
    assert lay.part_vertex_begin.tolist() == g["optimal_block_begin"]
    assert lay.halo_ids.size == 0
    check_layout(e, 6, part, 2, lay)


def test_fig_mot_layout():
    g = golden("fig_mot.json")
    e = np.array(g["topologies"]["star_plus_triangle"], np.int32)
    for sched, red in ((g["schedule_a"], 3), (g["schedule_b"], 1)):
        lay = O.remap(e, 6, np.array(sched, np.int32), 2)
        assert lay.halo_ids.size == red
        check_layout(e, 6, np.array(sched, np.int32), 2, lay)


@pytest.mark.parametrize("seed", range(25))
def test_random_layouts(seed):
    rng = np.random.default_rng(600 + seed)
    m, n = int(rng.integers(1, 120)), int(rng.integers(1, 60))
    n, e = S.random_multigraph(seed, m, n)
    k = int(rng.integers(1, 9))
    part = rng.integers(0, k, m).astype(np.int32)
    check_layout(e, n, part, k, O.remap(e, n, part, k))


def test_mesh_layout(small_mesh):
    M = small_mesh
    for P in (256, 1024):
        k = O.num_parts(M.m, P)
        for part in (O.partition(M.edges, M.n, P), O.default_partition(M.m, P)):
            check_layout(M.edges, M.n, part, k, O.remap(M.edges, M.n, part, k))


@pytest.mark.parametrize("seed", range(12))
def test_random_layouts_keyed(seed):
    """Reading Z22: with an order key (the partitioner's growth rank) the tasks of a
    partition are ordered by (key, id); every other step of O6 is unchanged."""
    rng = np.random.default_rng(900 + seed)
    m, n = int(rng.integers(1, 120)), int(rng.integers(1, 60))
    n, e = S.random_multigraph(70 + seed, m, n)
    k = int(rng.integers(1, 9))
    part = rng.integers(0, k, m).astype(np.int32)
    key = rng.integers(0, 5, m).astype(np.int32)          # ties broken by id
    check_layout(e, n, part, k, O.remap(e, n, part, k, key), key)


def test_mesh_layout_growth_order(small_mesh):
    """The growth-ranked remap of an EPG map keeps every invariant (L, C, bijection) and
    gives consecutive tasks of a partition shared or near vertices: the mean jump of the
    smaller local slot between consecutive tasks drops to less than half of the id order's
    (the staged kernel's threads then read nearby records)."""
    M = small_mesh
    P = 256
    k = O.num_parts(M.m, P)
    part, rank = O.partition(M.edges, M.n, P, method=2, ranked=True)
    lay_r = O.remap(M.edges, M.n, part, k, rank)
    check_layout(M.edges, M.n, part, k, lay_r, rank)
    lay_i = O.remap(M.edges, M.n, part, k)
    def jump(lay):
        d = []
        for p in range(k):
            sl = lay.slots[lay.part_edge_begin[p]:lay.part_edge_begin[p + 1]].astype(np.int64).min(axis=1)
            d.extend(np.abs(np.diff(sl)).tolist())
        return float(np.mean(d))
    assert jump(lay_r) < 0.5 * jump(lay_i)


def test_shard_halos(small_mesh):
    M = small_mesh
    P = 256
    k = O.num_parts(M.m, P)
    for G in (1, 2, 4, 8, k):
        part = O.partition(M.edges, M.n, P, G if G in (1, 2, 4, 8) else 1)
        lay = O.remap(M.edges, M.n, part, k)
        begin, ids = O.shard_halos(M.edges, M.n, part, k, G, lay.vertex_perm, lay.part_vertex_begin)
        if G == 1:
            assert ids.size == 0
        shard_of_part = np.zeros(k, np.int64)
        for g in range(G):
            shard_of_part[g * k // G:(g + 1) * k // G] = g
        # sum_g |Halo^g| = sum_v (#shards touching v - 1)
        touch = {}
        for (u, v), p in zip(M.edges.tolist(), part.tolist()):
            for x in (u, v):
                touch.setdefault(int(lay.vertex_perm[x]), set()).add(int(shard_of_part[p]))
        assert ids.size == sum(len(s) - 1 for s in touch.values())
        if G == k:
            assert ids.size == O.cost(M.edges, M.n, part, k).cut_cost
        pvb = lay.part_vertex_begin
        for g in range(G):
            for g2 in range(G):
                sl = ids[begin[g * G + g2]:begin[g * G + g2 + 1]]
                lo, hi = pvb[g2 * k // G], pvb[(g2 + 1) * k // G]
                assert np.all((sl >= lo) & (sl < hi)) and np.all(np.diff(sl) > 0)
                if sl.size:
                    assert g2 < g                         # halos flow from lower owners

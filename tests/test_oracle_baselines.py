"""Pins of the oracle's PowerGraph baselines (readings Z18, Z19 in DESIGN.md)."""
import numpy as np
import pytest

import oracle as O
import synth as S
from conftest import golden


@pytest.mark.parametrize("m,P,seed", [(1, 1, 0), (6, 3, 1), (1000, 64, 2), (1001, 100, 3), (4097, 4096, 4)])
def test_random_sizes_are_exact(m, P, seed):
    part = O.partition_random(m, P, seed)
    k = O.num_parts(m, P)
    assert np.array_equal(np.bincount(part, minlength=k), O.part_sizes(m, k))


@pytest.mark.parametrize("seed", [0, 1605, 2 ** 63 + 5])
def test_random_is_round_robin_over_the_splitmix_order(seed):
    """Pinned to synth.random_permutation, an independent (numpy argsort) construction of
    the same (SplitMix64(seed, e), e) order: the i-th edge of it lands in cluster i mod k."""
    m, P = 5000, 300
    k = O.num_parts(m, P)
    part = O.partition_random(m, P, seed)
    order = S.random_permutation(seed, m)
    assert np.array_equal(part[order], np.arange(m) % k)


def test_random_k1_and_seed_dependence():
    assert not O.partition_random(50, 4096, 9).any()
    a, b = O.partition_random(1000, 10, 1), O.partition_random(1000, 10, 2)
    assert not np.array_equal(a, b)
    assert np.array_equal(a, O.partition_random(1000, 10, 1))


def test_random_is_unbiased_on_two_triangle():
    """m = 6, k = 2: each edge lands in cluster 0 half the time over many seeds, and the
    mean cut cost exceeds the EP optimum (0) -- the paper's point."""
    g = golden("two_triangle.json")
    e = np.array(g["edges"], np.int32)
    parts = np.array([O.partition_random(6, 3, s) for s in range(2000)])
    freq = (parts == 0).mean(axis=0)
    assert np.all(np.abs(freq - 0.5) < 0.05)
    costs = [O.cost(e, 6, p, 2).cut_cost for p in parts[:500]]
    assert np.mean(costs) > 1.0 and min(costs) == 0


def test_greedy_spec_examples():
    # path of 4 edges, k = 2, capacity 2 -> {0,1} {2,3}, C = 1
    n, e = S.path_graph(4)
    p = O.partition_greedy(e, n, 2)
    assert p.tolist() == [0, 0, 1, 1]
    assert O.cost(e, n, p, 2).cut_cost == 1
    # m disjoint edges, k = m -> one edge per cluster, C = 0
    e = np.array([[2 * i, 2 * i + 1] for i in range(7)], np.int32)
    p = O.partition_greedy(e, 14, 1)
    assert sorted(p.tolist()) == list(range(7))
    assert O.cost(e, 14, p, 7).cut_cost == 0
    # two-triangle, interleaved order, k = 2 -> C = 0
    e = np.array([(0, 1), (3, 4), (1, 2), (4, 5), (0, 2), (3, 5)], np.int32)
    p = O.partition_greedy(e, 6, 3)
    assert O.cost(e, 6, p, 2).cut_cost == 0


def test_greedy_hand_traces():
    """Star K_{1,4}, P = 2 (k = 2, cap 2): e0 -> c0 (all scores 0, lowest id); e1 -> c0
    (holds 0); e2, e3 -> c1 (c0 full). Then m = 5, P = 2 (k = 3, cap 2):
    (0,1)->c0; (2,3)->c1 (scores 0: fewest edges, then lowest id); (0,2): c0 and c1 both
    score 1 with one edge each -> c0; (1,3): c0 full, c1 holds 3 -> c1; (4,5) -> c2."""
    star = np.array([(0, 1), (0, 2), (0, 3), (0, 4)], np.int32)
    p = O.partition_greedy(star, 5, 2)
    assert p.tolist() == [0, 0, 1, 1]
    assert O.cost(star, 5, p, 2).cut_cost == 1
    e = np.array([(0, 1), (2, 3), (0, 2), (1, 3), (4, 5)], np.int32)
    assert O.partition_greedy(e, 6, 2).tolist() == [0, 1, 0, 1, 2]


@pytest.mark.parametrize("seed", range(6))
def test_greedy_capacity_and_score_invariants(seed):
    """Every cluster holds <= ceil(m/k) edges; and each edge's cluster had the highest
    score among the clusters not full at that moment (replayed from the output)."""
    rng = np.random.default_rng(seed)
    m, nv = int(rng.integers(5, 400)), int(rng.integers(2, 60))
    n, e = S.random_multigraph(seed, m, nv)
    P = int(rng.integers(1, 40))
    k = O.num_parts(m, P)
    cap = -(-m // k)
    p = O.partition_greedy(e, n, P)
    assert np.bincount(p, minlength=k).max() <= cap
    present = [set() for _ in range(k)]
    size = [0] * k
    for i, (u, v) in enumerate(e):
        open_c = [c for c in range(k) if size[c] < cap]
        best = max((int(u in present[c]) + int(v in present[c])) for c in open_c)
        c = p[i]
        assert size[c] < cap and int(u in present[c]) + int(v in present[c]) == best
        present[c] |= {int(u), int(v)}
        size[c] += 1


def test_baselines_worse_than_ep_on_mesh(mesh_c1):
    """both baselines have significantly worse quality than the EP model; the
    random one is worse than the default schedule too."""
    M = mesh_c1
    P = 1024
    k = O.num_parts(M.m, P)
    c_ep = O.cost(M.edges, M.n, O.partition(M.edges, M.n, P), k).cut_cost
    c_def = O.cost(M.edges, M.n, O.default_partition(M.m, P), k).cut_cost
    c_rand = O.cost(M.edges, M.n, O.partition_random(M.m, P, 1605), k).cut_cost
    c_greedy = O.cost(M.edges, M.n, O.partition_greedy(M.edges, M.n, P), k).cut_cost
    assert c_ep < c_greedy and c_ep < c_rand
    assert c_rand > c_def

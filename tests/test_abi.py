"""CPU checks of the boundary: libepg.so loads, exports every symbol include/epg.h
declares, and its host EP partitioner (step a2, host C++) agrees with the oracle bit for
bit. No CUDA compute is called here."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
import synth as S
from conftest import ROOT, golden


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "epg.h")) as f:
        src = re.sub(r"/\*.*?\*/", "", f.read(), flags=re.S)
    return sorted(set(re.findall(r"\b(epg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1605_02043_b200 import epg
    lib = ctypes.CDLL(epg.LIB_PATH)
    declared = _declared_symbols()
    assert len(declared) >= 14
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(epg.SYMBOLS) == declared


def test_num_parts():
    from paper_1605_02043_b200 import epg
    for m, P in [(1, 1), (190245, 1024), (458168, 256), (10, 3)]:
        assert epg.num_parts(m, P) == O.num_parts(m, P)
    assert epg.num_parts(0, 5) == 0


def test_host_partition_fixtures():
    from paper_1605_02043_b200 import epg
    g = golden("fig_mot.json")
    e = np.array(g["topologies"]["star_plus_triangle"], np.int32)
    assert epg.partition_host(e, 6, 3).tolist() == g["schedule_b"]
    g2 = golden("two_triangle.json")
    assert epg.partition_host(np.array(g2["edges"], np.int32), 6, 3).tolist() == g2["optimal_partition"]


@pytest.mark.parametrize("seed", range(40))
def test_host_partition_random_bitexact(seed):
    from paper_1605_02043_b200 import epg
    rng = np.random.default_rng(900 + seed)
    m = int(rng.integers(1, 3000))
    n = int(rng.integers(1, 1500))
    n, e = S.random_multigraph(seed, m, n)
    P = int(rng.integers(1, 300))
    k = O.num_parts(m, P)
    for G in (1, 2, 4, 8):
        if G > k:
            continue
        assert np.array_equal(epg.partition_host(e, n, P, G), O.partition(e, n, P, G))


@pytest.mark.parametrize("P", [256, 1024, 4096])
def test_host_partition_mesh_bitexact(mesh_c1, P):
    from paper_1605_02043_b200 import epg
    M = mesh_c1
    assert np.array_equal(epg.partition_host(M.edges, M.n, P), O.partition(M.edges, M.n, P))


def test_host_partition_hierarchical_mesh(small_mesh):
    from paper_1605_02043_b200 import epg
    M = small_mesh
    for G in (2, 4, 8):
        assert np.array_equal(epg.partition_host(M.edges, M.n, 256, G), O.partition(M.edges, M.n, 256, G))


def test_host_partition_errors():
    from paper_1605_02043_b200 import epg
    with pytest.raises(epg.EpgError) as ex:
        epg.partition_host(np.array([[0, 1], [1, 7]], np.int32), 3, 2)
    assert ex.value.status == epg.ERR_INPUT and "edge 1" in ex.value.message
    with pytest.raises(epg.EpgError) as ex:
        epg.partition_host(np.array([[0, 1]], np.int32), 2, 4097)
    assert ex.value.status == epg.ERR_INFEASIBLE
    with pytest.raises(epg.EpgError) as ex:
        epg.partition_host(np.array([[0, 1]] * 4, np.int32), 2, 2, shards=4)
    assert ex.value.status == epg.ERR_INFEASIBLE
    with pytest.raises(epg.EpgError) as ex:
        epg.partition_host(np.zeros((0, 2), np.int32), 2, 2)
    assert ex.value.status == epg.ERR_INPUT


def test_host_partition_rmat_bitexact():
    """Hub vertices and parallel edges (R-MAT, Z15): many weight>1 edges of T."""
    from paper_1605_02043_b200 import epg
    n, e = S.rmat(10)
    for P, G in ((64, 1), (256, 1), (128, 4)):
        assert np.array_equal(epg.partition_host(e, n, P, G), O.partition(e, n, P, G))


@pytest.mark.parametrize("seed", range(12))
def test_baselines_bitexact(seed):
    """PowerGraph random / greedy baselines: library == oracle, bit for bit."""
    from paper_1605_02043_b200 import epg
    rng = np.random.default_rng(1200 + seed)
    m = int(rng.integers(1, 4000))
    nv = int(rng.integers(1, 800))
    n, e = S.random_multigraph(seed, m, nv)
    P = int(rng.integers(1, 200))
    assert np.array_equal(epg.partition_random_host(m, P, seed * 7919), O.partition_random(m, P, seed * 7919))
    assert np.array_equal(epg.partition_greedy_host(e, n, P), O.partition_greedy(e, n, P))


def test_baselines_bitexact_mesh_and_rmat(mesh_c1):
    from paper_1605_02043_b200 import epg
    M = mesh_c1
    for P in (256, 1024):
        assert np.array_equal(epg.partition_greedy_host(M.edges, M.n, P), O.partition_greedy(M.edges, M.n, P))
        assert np.array_equal(epg.partition_random_host(M.m, P, 1605), O.partition_random(M.m, P, 1605))
    n, e = S.rmat(11)
    assert np.array_equal(epg.partition_greedy_host(e, n, 128), O.partition_greedy(e, n, 128))


def test_baselines_errors():
    from paper_1605_02043_b200 import epg
    with pytest.raises(epg.EpgError) as ex:
        epg.partition_greedy_host(np.array([[0, 1], [1, 7]], np.int32), 3, 2)
    assert ex.value.status == epg.ERR_INPUT and "edge 1" in ex.value.message
    for bad in (0, 4097):
        with pytest.raises(epg.EpgError) as ex:
            epg.partition_random_host(10, bad)
        assert ex.value.status == epg.ERR_INFEASIBLE
    with pytest.raises(epg.EpgError) as ex:
        epg.partition_random_host(0, 4)
    assert ex.value.status == epg.ERR_INPUT


# ---------------------------------------------------------------- EPG-2 (O5', reading Z20)
def test_host_epg2_fixtures():
    from paper_1605_02043_b200 import epg
    g = golden("fig_mot.json")
    e = np.array(g["topologies"]["star_plus_triangle"], np.int32)
    assert epg.partition_host(e, 6, 3, method=epg.PARTITION_EPG2).tolist() == g["schedule_b"]
    g2 = golden("two_triangle.json")
    e2 = np.array(g2["edges"], np.int32)
    assert epg.partition_host(e2, 6, 3, method=epg.PARTITION_EPG2).tolist() == g2["optimal_partition"]


@pytest.mark.parametrize("seed", range(30))
def test_host_epg2_random_bitexact(seed):
    """Self-loops, parallel edges, isolated vertices, every shard count."""
    from paper_1605_02043_b200 import epg
    rng = np.random.default_rng(1900 + seed)
    m = int(rng.integers(1, 3000))
    n = int(rng.integers(1, 1500))
    n, e = S.random_multigraph(300 + seed, m, n)
    P = int(rng.integers(1, 300))
    k = O.num_parts(m, P)
    for G in (1, 2, 4, 8):
        if G > k:
            continue
        assert np.array_equal(epg.partition_host(e, n, P, G, method=epg.PARTITION_EPG2),
                              O.partition(e, n, P, G, method=2))


@pytest.mark.parametrize("P", [256, 1024])
def test_host_epg2_mesh_and_rmat_bitexact(mesh_c1, P):
    from paper_1605_02043_b200 import epg
    M = mesh_c1
    assert np.array_equal(epg.partition_host(M.edges, M.n, P, method=epg.PARTITION_EPG2),
                          O.partition(M.edges, M.n, P, method=2))
    n, e = S.rmat(10)
    assert np.array_equal(epg.partition_host(e, n, P // 4, 2, method=epg.PARTITION_EPG2),
                          O.partition(e, n, P // 4, 2, method=2))


def test_host_partition_method_errors():
    from paper_1605_02043_b200 import epg
    with pytest.raises(epg.EpgError) as ex:
        epg.partition_host(np.array([[0, 1]], np.int32), 2, 1, method=3)
    assert ex.value.status == epg.ERR_INPUT


@pytest.mark.parametrize("method", [1, 2])
def test_host_ranked_matches_oracle(method, mesh_c1):
    """epg_partition_host_ranked: the growth step of every task (reading Z22) equals the
    oracle's, flat and hierarchical, on random multigraphs and the C1 mesh."""
    from paper_1605_02043_b200 import epg
    for seed in range(8):
        rng = np.random.default_rng(4400 + seed)
        m, n0 = int(rng.integers(5, 400)), int(rng.integers(3, 120))
        n, e = S.random_multigraph(4500 + seed, m, n0)
        P = int(rng.integers(2, 40))
        for shards in (1, 2):
            if shards > O.num_parts(m, P):
                continue
            part, rank = epg.partition_host_ranked(e, n, P, shards, method)
            rp, rr = O.partition(e, n, P, shards, method=method, ranked=True)
            assert np.array_equal(part, rp) and np.array_equal(rank, rr)
    part, rank = epg.partition_host_ranked(mesh_c1.edges, mesh_c1.n, 1024, 1, method)
    rp, rr = O.partition(mesh_c1.edges, mesh_c1.n, 1024, method=method, ranked=True)
    assert np.array_equal(part, rp) and np.array_equal(rank, rr)

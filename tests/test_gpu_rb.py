"""GPU: the library's EPG-RB partitioner (GPU bisection levels + EPG-2 leaves on the host
cores; include/epg.h EPG_PARTITION_RB, reading Z21) equals the oracle's plain sequential
transcription (orc_partition_rb) bit for bit, and its load report equals the oracle's
Eq. (1) cost of that map."""
import numpy as np
import pytest
import torch

import oracle as O
import synth as S
from conftest import golden

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _check(ctx, e, n, P, shards, lp, host_edges=False):
    k = O.num_parts(len(e), P)
    edges = torch.from_numpy(np.ascontiguousarray(e)) if host_edges else dev(e)
    out = torch.empty(len(e), dtype=torch.int32, device=edges.device)
    part, rank, rep = ctx.partition_rb(edges, n, P, shards, lp, out=out, ranked=True)
    ref, ref_rank = O.partition_rb(e, n, P, shards, lp, ranked=True)
    assert np.array_equal(part.cpu().numpy(), ref)
    assert np.array_equal(rank.cpu().numpy(), ref_rank)          # growth steps (reading Z22)
    r = O.cost(e, n, ref, k)
    assert (rep.load_count, rep.cut_cost, rep.touched, rep.max_size, rep.min_size) == \
        (r.load_count, r.cut_cost, r.touched, r.max_size, r.min_size)
    return rep


def test_rb_fig_mot():
    from paper_1605_02043_b200 import epg
    ctx = epg.Context(0)
    g = golden("fig_mot.json")
    for topo in g["topologies"].values():
        e = np.array(topo, np.int32)
        rep = _check(ctx, e, int(e.max()) + 1, 3, 1, 1)
        assert rep.load_count == 7


@pytest.mark.parametrize("seed", range(10))
def test_rb_random_multigraphs(seed):
    from paper_1605_02043_b200 import epg
    ctx = epg.Context(0)
    rng = np.random.default_rng(9100 + seed)
    m, n0 = int(rng.integers(20, 3000)), int(rng.integers(5, 800))
    n, e = S.random_multigraph(900 + seed, m, n0)
    P = int(rng.integers(2, 64))
    k = O.num_parts(m, P)
    for shards in (1, 2, 4, 8):
        if shards > k:
            continue
        for lp in (1, 3):
            _check(ctx, e, n, P, shards, lp, host_edges=(seed % 2 == 1))


@pytest.mark.parametrize("shards", [1, 4])
def test_rb_c1(mesh_c1, shards):
    from paper_1605_02043_b200 import epg
    ctx = epg.Context(0)
    rep = _check(ctx, mesh_c1.edges, mesh_c1.n, 1024, shards, 16)
    assert rep.replication < 1.25


def test_rb_rmat_hubs():
    """R-MAT (power-law, hubs above 4P tasks carry no BFS adjacency), scale 12, P = 64."""
    from paper_1605_02043_b200 import epg
    ctx = epg.Context(0)
    n, e = S.rmat(12)
    _check(ctx, e, n, 64, 1, 8)
    _check(ctx, e, n, 64, 2, 8)


def test_rb_method_on_context(small_mesh):
    """epg_set_partition_method(EPG_PARTITION_RB): epg_partition uses it (leaf_parts 512 or
    EPG_RB_LEAF_PARTS); the host-only entry point rejects it."""
    from paper_1605_02043_b200 import epg
    M = small_mesh
    ctx = epg.Context(0)
    ctx.set_partition_method(epg.PARTITION_RB)
    part, rep = ctx.partition(dev(M.edges), M.n, 16)
    assert np.array_equal(part.cpu().numpy(), O.partition_rb(M.edges, M.n, 16, 1, 512))
    with pytest.raises(epg.EpgError) as ex:
        epg.partition_host(M.edges, M.n, 16, method=epg.PARTITION_RB)
    assert ex.value.status == epg.ERR_INPUT
    with pytest.raises(epg.EpgError) as ex:
        ctx.partition_rb(dev(M.edges), M.n, 16, 1, 0)
    assert ex.value.status == epg.ERR_INPUT

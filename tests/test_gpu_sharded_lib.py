"""GPU: the library's sharded step (epg_run_sharded / epg_run_sharded_group, SURVEY §8(b)
epg_comm_init and §8(e)): the O7 halo exchange (pull rows, edge kernel over the shard's
partitions, push partial sums, finalise) inside libepg.so.

* G = 2, 4, 8 members of an in-process group on one GPU (epg_comm_init_local: the same
  exchange schedule as NCCL, transfers as device copies): the authoritative (owned) rows of
  all members together equal the fp64 oracle within the Z14 tolerance (cfd) and bit for bit
  (integer-valued gather-scatter), and equal the single-GPU epg_run within fp32 rounding;
* a one-rank NCCL communicator (epg_comm_unique_id + epg_comm_init, nranks = 1) runs the
  same path with the NCCL transport: bit-identical to epg_run over several steps;
* every group test runs with both pushes: the sequential schedule and the fused peer push
  (EPG_EXCHANGE=p2p, atomics into the owners' accumulators: integer-valued gather-scatter still
  exact, cfd within the tolerance).
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth as S

pytestmark = pytest.mark.gpu

TOL = 1e-5


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def normwise_err(got, ref):
    got = np.asarray(got, np.float64).reshape(ref.shape[0], -1)
    ref = np.asarray(ref, np.float64).reshape(ref.shape[0], -1)
    return np.abs(got - ref).max(axis=0) / np.maximum(np.abs(ref).max(axis=0), 1e-300)


def _group(G, edges, n, P):
    from paper_1605_02043_b200 import epg
    ctxs = [epg.Context(0) for _ in range(G)]
    E = dev(edges)
    part, rep = ctxs[0].partition_rb(E, n, P, shards=G, leaf_parts=8)
    k = epg.num_parts(len(edges), P)
    layouts, plans = zip(*[c.remap(E, n, part, k, halo_cap=rep.cut_cost) for c in ctxs])
    epg.comm_init_local(ctxs)
    return ctxs, list(layouts), list(plans), part


def _owned(ctx, plan, G, g, out):
    r = ctx.shard_ranges(plan, G, g)
    lo, hi = r["vertex_first"], r["vertex_first"] + r["vertex_count"]
    return lo, hi, out[lo:hi].cpu().numpy()


@pytest.fixture(params=["nccl-schedule", "p2p"])
def exchange_mode(request, monkeypatch):
    """The push of the exchange: the sequential schedule (partials reduced, sent, accumulated in a
    fixed order) or the fused peer push (EPG_EXCHANGE=p2p: the boundary edge kernel adds each
    foreign partial into its owner's accumulator; in the in-process group the members'
    accumulators are the peer memory)."""
    if request.param == "p2p":
        monkeypatch.setenv("EPG_EXCHANGE", "p2p")
    else:
        monkeypatch.delenv("EPG_EXCHANGE", raising=False)
    return request.param


@pytest.mark.parametrize("G", [2, 4, 8])
def test_group_cfd_step(mesh_c1, G, exchange_mode):
    from paper_1605_02043_b200 import epg
    M = mesh_c1
    ctxs, Ls, plans, part = _group(G, M.edges, M.n, 256)
    U, dt = S.cfd_state(M.n), S.cfd_dt(M.volume)
    L = Ls[0]
    vp = L.vertex_perm
    states, outs = [], []
    for c, Lg in zip(ctxs, Ls):
        a = c.permute_rows(dev(U), Lg.vertex_perm, epg.PERM_SCATTER)
        b = torch.empty_like(a)
        nrm = c.permute_rows(dev(M.normals), Lg.edge_perm, epg.PERM_GATHER)
        d = c.permute_rows(dev(dt), Lg.vertex_perm, epg.PERM_SCATTER)
        states.append((a, b, nrm, d))
        outs.append(b)
    epg.run_sharded_group(ctxs, plans, epg.KERNEL_CFD_FLUX, states)
    torch.cuda.synchronize()
    full = np.zeros((M.n, 5), np.float32)
    covered = 0
    for g in range(G):
        lo, hi, rows = _owned(ctxs[g], plans[g], G, g, outs[g])
        full[lo:hi] = rows
        covered += hi - lo
    # untouched rows (copied by every member) complete the state
    t = plans[0].touched
    full[t:] = outs[0][t:].cpu().numpy()
    assert covered == t
    got = full[vp.cpu().numpy()]                       # original vertex order
    ref, _ = O.cfd_step(M.edges, M.n, M.normals, U, dt)
    assert normwise_err(got, ref).max() <= TOL
    # the single-GPU step on the same map
    c1 = epg.Context(0)
    L1, p1 = c1.remap(dev(M.edges), M.n, part, epg.num_parts(M.m, 256))
    a = c1.permute_rows(dev(U), L1.vertex_perm, epg.PERM_SCATTER)
    b = torch.empty_like(a)
    c1.run(p1, epg.KERNEL_CFD_FLUX, a, b, c1.permute_rows(dev(M.normals), L1.edge_perm, epg.PERM_GATHER),
           c1.permute_rows(dev(dt), L1.vertex_perm, epg.PERM_SCATTER), 1)
    single = c1.permute_rows(b, L1.vertex_perm, epg.PERM_GATHER).cpu().numpy()
    assert normwise_err(got, single.astype(np.float64)).max() <= 1e-6


@pytest.mark.parametrize("G", [2, 8])
def test_group_gather_scatter_exact(G, exchange_mode):
    from paper_1605_02043_b200 import epg
    n, e = S.rmat(13)
    ctxs, Ls, plans, part = _group(G, e, n, 128)
    x = S.int_vector(3, n, 0, 7)
    states, outs = [], []
    for c, Lg in zip(ctxs, Ls):
        a = c.permute_rows(dev(x), Lg.vertex_perm, epg.PERM_SCATTER)
        b = torch.empty_like(a)
        states.append((a, b, None, None))
        outs.append(b)
    epg.run_sharded_group(ctxs, plans, epg.KERNEL_GATHER_SCATTER, states)
    full = np.zeros(n, np.float32)
    for g in range(G):
        lo, hi, rows = _owned(ctxs[g], plans[g], G, g, outs[g])
        full[lo:hi] = rows
    got = full[Ls[0].vertex_perm.cpu().numpy()]
    assert np.array_equal(got.astype(np.float64), O.gather_scatter(e, n, x))


def test_nccl_one_rank_matches_epg_run(small_mesh):
    from paper_1605_02043_b200 import epg
    M = small_mesh
    ctx = epg.Context(0)
    ctx.comm_init(epg.comm_unique_id(), 1, 0)
    E = dev(M.edges)
    part, rep = ctx.partition(E, M.n, 256)
    L, plan = ctx.remap(E, M.n, part, epg.num_parts(M.m, 256))
    U, dt = S.cfd_state(M.n), S.cfd_dt(M.volume)
    a = ctx.permute_rows(dev(U), L.vertex_perm, epg.PERM_SCATTER)
    nrm = ctx.permute_rows(dev(M.normals), L.edge_perm, epg.PERM_GATHER)
    d = ctx.permute_rows(dev(dt), L.vertex_perm, epg.PERM_SCATTER)
    x1, y1 = a.clone(), torch.empty_like(a)
    r1 = ctx.run_sharded(plan, epg.KERNEL_CFD_FLUX, x1, y1, nrm, d, 3)
    x2, y2 = a.clone(), torch.empty_like(a)
    r2 = ctx.run(plan, epg.KERNEL_CFD_FLUX, x2, y2, nrm, d, 3)
    assert np.array_equal(r1.cpu().numpy(), r2.cpu().numpy())

"""GPU: the launch-path features of epg_run (include/epg.h) must not change results.

* multi-wave grids (more execution partitions than resident CTAs) bulk-prefetch the next
  wave's ranges into L2 (EPG_PREFETCH_AHEAD) -- bit-identical to no prefetch, and within
  the Z14 tolerance of the fp64 oracle;
* the occupancy path replays a cached CUDA graph per (plan, kernel, buffers, steps)
  (EPG_GRAPHS) -- bit-identical to direct launches, for several buffer pairs and step
  counts reusing the cache, including after the cache is evicted (> 16 entries)."""
import os

import numpy as np
import pytest
import torch

import oracle as O
import synth as S

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _prep(M, P, method=2):
    from paper_1605_02043_b200 import epg
    ctx = epg.Context(0)
    ctx.set_partition_method(method)
    part, _ = ctx.partition(dev(M.edges), M.n, P)
    L, plan = ctx.remap(dev(M.edges), M.n, part, epg.num_parts(M.m, P))
    U, dt = S.cfd_state(M.n), S.cfd_dt(M.volume)
    Un = ctx.permute_rows(dev(U), L.vertex_perm, epg.PERM_SCATTER)
    nrm = ctx.permute_rows(dev(M.normals), L.edge_perm, epg.PERM_GATHER)
    dtn = ctx.permute_rows(dev(dt), L.vertex_perm, epg.PERM_SCATTER)
    return ctx, L, plan, U, dt, Un, nrm, dtn


def _env(name, value):
    old = os.environ.get(name)
    if value is None:
        os.environ.pop(name, None)
    else:
        os.environ[name] = value
    return old


def test_multiwave_prefetch_bitexact_and_oracle():
    from paper_1605_02043_b200 import epg
    M = S.config_mesh("c1")
    ctx, L, plan, U, dt, Un, nrm, dtn = _prep(M, 32)
    assert plan.k_exec > 148 * 4                   # more partitions than one resident wave
    outs = {}
    for ahead in ("0", None):                      # prefetch off, then the default (one wave ahead)
        old = _env("EPG_PREFETCH_AHEAD", ahead)
        try:
            o = torch.empty_like(Un)
            ctx.run(plan, epg.KERNEL_CFD_FLUX, Un, o, nrm, dtn, 1)
            outs[ahead] = o.cpu().numpy()
        finally:
            _env("EPG_PREFETCH_AHEAD", old)
    assert np.array_equal(outs["0"], outs[None])
    got = np.empty_like(outs[None])
    got[:] = outs[None][L.vertex_perm.cpu().numpy()]   # back to the original vertex order
    ref, _ = O.cfd_step(M.edges, M.n, M.normals, U, dt)
    err = np.abs(got - ref).max(axis=0) / np.abs(ref).max(axis=0)
    assert err.max() <= 1e-5


def test_graph_replay_bitexact():
    from paper_1605_02043_b200 import epg
    M = S.kuhn_mesh(nbox=12, n_keep=9000)
    ctx, L, plan, U, dt, Un, nrm, dtn = _prep(M, 256)
    pairs = [(Un.clone(), torch.empty_like(Un)) for _ in range(3)]

    def sweep():
        res = []
        for rep in range(7):                       # 3 buffer pairs x 3 step counts: 9 cache keys
            for j, (a, b) in enumerate(pairs):
                for steps in (1, 2, 3):
                    a.copy_(Un)
                    out = ctx.run(plan, epg.KERNEL_CFD_FLUX, a, b, nrm, dtn, steps)
                    res.append(out.cpu().numpy())
        return res

    old = _env("EPG_GRAPHS", "0")
    try:
        direct = sweep()
        _env("EPG_GRAPHS", "2")                    # one-step calls through graphs too
        graphed = sweep()
        # more than 16 keys: the cache is evicted and rebuilt, results unchanged
        extra = [(Un.clone(), torch.empty_like(Un)) for _ in range(8)]
        for a, b in extra:
            for steps in (1, 2):
                a.copy_(Un)
                out = ctx.run(plan, epg.KERNEL_CFD_FLUX, a, b, nrm, dtn, steps)
                assert np.array_equal(out.cpu().numpy(), graphed[steps - 1])
    finally:
        _env("EPG_GRAPHS", old)
    default = sweep()                              # default: graphs for steps >= 2 only
    for x, y, z in zip(direct, graphed, default):
        assert np.array_equal(x, y) and np.array_equal(x, z)


@pytest.mark.timeout(300, method="thread")
def test_pipelined_variant_one_plan_two_grids():
    """the persistent pipelined kernel (variant 2) synchronises its CTAs on a
    per-plan monotone counter. Its grid (SMs x occupancy) depends on the functor's shared
    memory, so one plan run alternately with the cfd functor and with gather-scatter
    launches different grids in turn; the barrier target must follow the cumulative
    arrivals (no deadlock, no early release -- both results stay correct)."""
    from paper_1605_02043_b200 import epg
    M = S.config_mesh("c1")
    P = 64
    ctx = epg.Context(0)
    ctx.set_variant(2)
    ctx.set_partition_method(2)
    E = dev(M.edges)
    part, _ = ctx.partition(E, M.n, P)
    L, plan = ctx.remap(E, M.n, part, epg.num_parts(M.m, P))
    U, dt = S.cfd_state(M.n), S.cfd_dt(M.volume)
    Un = ctx.permute_rows(dev(U), L.vertex_perm, epg.PERM_SCATTER)
    nrm = ctx.permute_rows(dev(M.normals), L.edge_perm, epg.PERM_GATHER)
    dtn = ctx.permute_rows(dev(dt), L.vertex_perm, epg.PERM_SCATTER)
    ref_cfd, _ = O.cfd_step(M.edges, M.n, M.normals, U, dt)
    x = S.int_vector(5, M.n, 0, 7)
    ref_gs = O.gather_scatter(M.edges, M.n, x)
    xn = ctx.permute_rows(dev(x), L.vertex_perm, epg.PERM_SCATTER)
    for rep in range(3):
        o = torch.empty_like(Un)
        ctx.run(plan, epg.KERNEL_CFD_FLUX, Un, o, nrm, dtn, 1)
        got = ctx.permute_rows(o, L.vertex_perm, epg.PERM_GATHER).cpu().numpy()
        assert (np.abs(got - ref_cfd).max(axis=0) / np.abs(ref_cfd).max(axis=0)).max() <= 1e-5
        y = torch.empty_like(xn)
        ctx.run(plan, epg.KERNEL_GATHER_SCATTER, xn, y, None, None, 1)
        got = ctx.permute_rows(y, L.vertex_perm, epg.PERM_GATHER).cpu().numpy()
        assert np.array_equal(got.astype(np.float64), ref_gs)


@pytest.mark.parametrize("cfg,P", [("c1", 1032), ("c2", 1032), ("c1", 1100)])
def test_wide_cta_instance(cfg, P):
    """Partitions of 1025..1152 edges run on the 288-thread (9-warp) instance of the edge
    kernel (bench.py's SM-balanced C2 size P = 1032): growth-ordered EPG-RB map as in the
    bench, exec limits (1152 rows, 1152 edges); within the Z14 tolerance of the fp64 oracle,
    normwise and componentwise, and the same result through epg_run(steps=2) (graph) as
    through two one-step calls (direct launches)."""
    from paper_1605_02043_b200 import epg
    M = S.config_mesh(cfg)
    ctx = epg.Context(0)
    ctx.set_exec_limits(1152, 1152)
    E = dev(M.edges)
    part, rank, _ = ctx.partition_rb(E, M.n, P, ranked=True)
    k = epg.num_parts(M.m, P)
    L, plan = ctx.remap(E, M.n, part, k, order_key=rank)
    assert plan.k_exec == k                       # no execution splits: every partition fits
    U, dt = S.cfd_state(M.n), S.cfd_dt(M.volume)
    Un = ctx.permute_rows(dev(U), L.vertex_perm, epg.PERM_SCATTER)
    nrm = ctx.permute_rows(dev(M.normals), L.edge_perm, epg.PERM_GATHER)
    dtn = ctx.permute_rows(dev(dt), L.vertex_perm, epg.PERM_SCATTER)
    out = torch.empty_like(Un)
    ctx.run(plan, epg.KERNEL_CFD_FLUX, Un, out, nrm, dtn, 1)
    got = ctx.permute_rows(out, L.vertex_perm, epg.PERM_GATHER).cpu().numpy().astype(np.float64)
    ref, _ = O.cfd_step(M.edges, M.n, M.normals, U, dt)
    err = np.abs(got - ref).max(axis=0) / np.abs(ref).max(axis=0)
    assert err.max() <= 1e-5
    S_v = O.cfd_flux_abs(M.edges, M.n, M.normals, U)
    comp = np.abs(got - ref) / np.maximum(np.abs(ref), dt[:, None] * S_v)
    assert comp.max() <= 1e-5
    a, b = Un.clone(), torch.empty_like(Un)
    ctx.run(plan, epg.KERNEL_CFD_FLUX, a, b, nrm, dtn, 1)
    ctx.run(plan, epg.KERNEL_CFD_FLUX, b, a, nrm, dtn, 1)
    c, d = Un.clone(), torch.empty_like(Un)
    two = ctx.run(plan, epg.KERNEL_CFD_FLUX, c, d, nrm, dtn, 2)
    assert np.array_equal(a.cpu().numpy(), two.cpu().numpy())


@pytest.mark.parametrize("cfg,P", [("c1", 1024), ("c1", 256)])
def test_plan_options_bitexact(cfg, P):
    """Execution-plan choices that must not change a single result bit (include/epg.h):
    the bank-conflict-aware record placement (EPG_PLACE=0: identity positions) and the 16-byte
    finalise records (EPG_FIN_REC16=0: the 32-byte records) -- each plan built under the option,
    two cfd steps, compared bit for bit with the default plan; and the default within the Z14
    tolerance of the fp64 oracle."""
    from paper_1605_02043_b200 import epg
    M = S.config_mesh(cfg)
    U, dt = S.cfd_state(M.n), S.cfd_dt(M.volume)
    E = dev(M.edges)
    ctx = epg.Context(0)
    part, rank, _ = ctx.partition_rb(E, M.n, P, ranked=True)
    k = epg.num_parts(M.m, P)

    def run(env):
        olds = {kk: _env(kk, vv) for kk, vv in env.items()}
        try:
            L, plan = ctx.remap(E, M.n, part, k, order_key=rank)
        finally:
            for kk, vv in olds.items():
                _env(kk, vv)
        Un = ctx.permute_rows(dev(U), L.vertex_perm, epg.PERM_SCATTER)
        nrm = ctx.permute_rows(dev(M.normals), L.edge_perm, epg.PERM_GATHER)
        dtn = ctx.permute_rows(dev(dt), L.vertex_perm, epg.PERM_SCATTER)
        out = ctx.run(plan, epg.KERNEL_CFD_FLUX, Un, torch.empty_like(Un), nrm, dtn, 2)
        return ctx.permute_rows(out, L.vertex_perm, epg.PERM_GATHER).cpu().numpy()

    base = run({})
    assert np.array_equal(base, run({"EPG_PLACE": "0"}))
    assert np.array_equal(base, run({"EPG_FIN_REC16": "0"}))
    ref, _ = O.cfd_step(M.edges, M.n, M.normals, U, dt)
    ref2, _ = O.cfd_step(M.edges, M.n, M.normals, ref.astype(np.float32), dt)
    err = np.abs(base - ref2).max(axis=0) / np.abs(ref2).max(axis=0)
    assert err.max() <= 2e-5


def test_run_edges_one_wave_chain_equals_run():
    """One-wave epg_run_edges launches trigger their PDL dependents at the start, so the next
    launch's plan-data prologue overlaps them: chains of run_edges + run_finalise over two
    replicas (own plans and buffers, one context stream), issued back to back for three
    rounds, give epg_run's result bit for bit (the dependent still waits before it reads state)."""
    from paper_1605_02043_b200 import epg
    M = S.config_mesh("c1")
    ctx, L, plan, U, dt, Un, nrm, dtn = _prep(M, 1024)
    assert plan.k_exec <= 148 * 4                # one resident wave
    part, _ = ctx.partition(dev(M.edges), M.n, 1024)
    L2, plan2 = ctx.remap(dev(M.edges), M.n, part, epg.num_parts(M.m, 1024))   # a second replica
    reps = [(plan, Un, nrm, dtn),
            (plan2, ctx.permute_rows(dev(U), L2.vertex_perm, epg.PERM_SCATTER),
             ctx.permute_rows(dev(M.normals), L2.edge_perm, epg.PERM_GATHER),
             ctx.permute_rows(dev(dt), L2.vertex_perm, epg.PERM_SCATTER))]
    chain, ref = [], []
    for pl, u, nr, dd in reps:
        chain.append([pl, u.clone(), torch.empty_like(u), nr, dd])
        ref.append(ctx.run(pl, epg.KERNEL_CFD_FLUX, u.clone(), torch.empty_like(u), nr, dd, 3).clone())
    for _ in range(3):
        for c in chain:
            pl, a, b, nr, dd = c
            ctx.run_edges(pl, epg.KERNEL_CFD_FLUX, a, b, nr, dd)
            ctx.run_finalise(pl, epg.KERNEL_CFD_FLUX, a, b, nr, dd)
            c[1], c[2] = b, a
    torch.cuda.synchronize()
    for c, r in zip(chain, ref):
        assert torch.equal(c[1], r)


def test_prewait_prefetch_bitexact():
    """Single-wave grids L2-prefetch their state rows before the PDL wait (EPG_PREWAIT_PF, on by
    default): a hint only -- the results with and without it are identical, and equal epg_run's
    multi-step call whose later steps skip it."""
    from paper_1605_02043_b200 import epg
    M = S.config_mesh("c1")
    ctx, L, plan, U, dt, Un, nrm, dtn = _prep(M, 1024)
    assert plan.k_exec <= 148 * 4
    outs = {}
    for pf in ("0", "1"):
        old = _env("EPG_PREWAIT_PF", pf)
        try:
            a, b = Un.clone(), torch.empty_like(Un)
            for _ in range(2):                     # two one-step calls (each a first step)
                ctx.run(plan, epg.KERNEL_CFD_FLUX, a, b, nrm, dtn, 1)
                a, b = b, a
            torch.cuda.synchronize()
            outs[pf] = a.clone()
        finally:
            _env("EPG_PREWAIT_PF", old)
    assert torch.equal(outs["0"], outs["1"])
    two = ctx.run(plan, epg.KERNEL_CFD_FLUX, Un.clone(), torch.empty_like(Un), nrm, dtn, 2)
    assert torch.equal(two, outs["1"])

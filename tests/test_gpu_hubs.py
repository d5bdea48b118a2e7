"""Hub split: shared vertices with many halo entries are reduced
through a per-hub accumulator (one red.global.add per execution partition and hub)
instead of the gathered finalise. Same results as the oracle: bit-exact for
integer-valued data (every fp32 partial sum is exact, so the order does not matter),
within the Z14 tolerance otherwise."""
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
    return (np.abs(got - ref).max(axis=0) / np.maximum(np.abs(ref).max(axis=0), 1e-300))


def _ctx(hub_min, variant=3):
    from paper_1605_02043_b200 import epg
    c = epg.Context(0)
    c.set_variant(variant)
    c.set_hub_split(hub_min)
    return c


def _scalar(ctx, kernel, e, n, part, k, x, w=None, steps=1):
    from paper_1605_02043_b200 import epg
    L, plan = ctx.remap(dev(e), n, dev(part), k)
    xn = ctx.permute_rows(dev(x), L.vertex_perm, epg.PERM_SCATTER)
    wn = None if w is None else ctx.permute_rows(dev(w), L.edge_perm, epg.PERM_GATHER)
    out = torch.empty_like(xn)
    res = ctx.run(plan, kernel, xn, out, wn, steps=steps)
    return ctx.permute_rows(res, L.vertex_perm, epg.PERM_GATHER).cpu().numpy(), plan


@pytest.fixture(scope="module")
def rmat14():
    n, e = S.rmat(14)
    P = 512
    return n, e, P, O.partition(e, n, P)


@pytest.mark.parametrize("hub_min", [0, 1, 2, 7, 33])
def test_rmat_hub_split_integer_exact(rmat14, hub_min):
    from paper_1605_02043_b200 import epg
    n, e, P, part = rmat14
    x = S.int_vector(1608, n, 0, 7)
    got, plan = _scalar(_ctx(hub_min), epg.KERNEL_GATHER_SCATTER, e, n, part, O.num_parts(len(e), P), x)
    assert np.array_equal(got.astype(np.float64), O.gather_scatter(e, n, x))
    assert plan.hub_min == hub_min
    if hub_min == 0:
        assert plan.hubs == 0
    else:
        assert 0 < plan.hubs <= plan.shared
    if hub_min == 1:
        assert plan.hubs == plan.shared           # every shared vertex has >= 1 halo entry


def test_rmat_hub_split_two_steps_exact(rmat14):
    """The accumulator is cleared by the hub finalise: step 2 sees no leftovers."""
    from paper_1605_02043_b200 import epg
    n, e, P, part = rmat14
    x = S.int_vector(1610, n, 0, 3)
    got, plan = _scalar(_ctx(2), epg.KERNEL_GATHER_SCATTER, e, n, part, O.num_parts(len(e), P), x, steps=2)
    assert plan.hubs > 0
    ref = O.gather_scatter(e, n, O.gather_scatter(e, n, x))
    assert ref.max() < 2 ** 24                    # every partial sum exact in fp32
    assert np.array_equal(got.astype(np.float64), ref)


def test_rmat_hub_split_float_tolerance(rmat14):
    from paper_1605_02043_b200 import epg
    n, e, P, part = rmat14
    x = S.uniform01(1611, np.arange(n, dtype=np.uint64)).astype(np.float32)
    got, plan = _scalar(_ctx(2), epg.KERNEL_GATHER_SCATTER, e, n, part, O.num_parts(len(e), P), x)
    assert plan.hubs > 0
    assert normwise_err(got, O.gather_scatter(e, n, x)).max() <= TOL


def test_cfd_default_has_no_hubs_and_forced_hubs_match(small_mesh):
    """cfd meshes (degree <= 4) have no hubs at the default; forcing every shared vertex
    through the accumulator (hub_min = 1, five reds per row) still matches the oracle."""
    from paper_1605_02043_b200 import epg
    M = small_mesh
    P = 512
    part = O.partition(M.edges, M.n, P)
    k = O.num_parts(M.m, P)
    U = S.cfd_state(M.n)
    dt = S.cfd_dt(M.volume).astype(np.float32)
    ref, _ = O.cfd_step(M.edges, M.n, M.normals, U, dt)
    for hub_min, expect_hubs in ((-1, False), (1, True)):
        ctx = _ctx(hub_min)
        L, plan = ctx.remap(dev(M.edges), M.n, dev(part), k)
        assert (plan.hubs > 0) == expect_hubs
        Un = ctx.permute_rows(dev(U), L.vertex_perm, epg.PERM_SCATTER)
        nrm = ctx.permute_rows(dev(M.normals), L.edge_perm, epg.PERM_GATHER)
        dtn = ctx.permute_rows(dev(dt), L.vertex_perm, epg.PERM_SCATTER)
        out = torch.empty_like(Un)
        ctx.run(plan, epg.KERNEL_CFD_FLUX, Un, out, nrm, dtn)
        got = ctx.permute_rows(out, L.vertex_perm, epg.PERM_GATHER).cpu().numpy()
        assert normwise_err(got, ref).max() <= TOL


def test_stencil_spmv_hub_split_exact():
    from paper_1605_02043_b200 import epg
    n, e, w = S.stencil2d_spmv(120)
    N = n // 2
    x = np.concatenate([S.int_vector(1609, N, -8, 8), np.zeros(N, np.float32)])
    P = 1024
    part = O.partition(e, n, P)
    got, plan = _scalar(_ctx(1), epg.KERNEL_SPMV, e, n, part, O.num_parts(len(e), P), x, w)
    assert plan.hubs > 0
    assert np.array_equal(got.astype(np.float64), O.spmv(e, n, w, x))


@pytest.mark.parametrize("variant", [1, 2])
def test_other_variants_ignore_hubs(rmat14, variant):
    """Variants 1 and 2 have their own finalise over every halo entry; a hub plan is
    still exact through them."""
    from paper_1605_02043_b200 import epg
    n, e, P, part = rmat14
    x = S.int_vector(1612, n, 0, 7)
    ctx = _ctx(2, variant)
    try:
        got, plan = _scalar(ctx, epg.KERNEL_GATHER_SCATTER, e, n, part, O.num_parts(len(e), P), x)
    except epg.EpgError as ex:                    # variant 2 may not fit the plan
        assert variant == 2 and ex.status == epg.ERR_INFEASIBLE
        return
    assert plan.hubs > 0
    assert np.array_equal(got.astype(np.float64), O.gather_scatter(e, n, x))


def test_shards_with_hub_plan_exact():
    """The shard path (run_edges / run_finalise) on a plan whose blobs carry hub indices:
    it sums every halo partial through hv_list, so it stays exact."""
    from paper_1605_02043_b200 import epg
    from paper_1605_02043_b200.shard import Shard, run_virtual, assemble_owned
    n, e = S.rmat(13)
    x = S.int_vector(9, n, 0, 7)
    P, G = 512, 4
    k = O.num_parts(e.shape[0], P)
    ctx = _ctx(2)
    E = dev(e)
    part, _ = ctx.partition(E, n, P, shards=G)
    L, plan = ctx.remap(E, n, part, k)
    assert plan.hubs > 0
    xn = ctx.permute_rows(dev(x), L.vertex_perm, epg.PERM_SCATTER)
    shards = [Shard(ctx, plan, L, epg.KERNEL_GATHER_SCATTER, G, g) for g in range(G)]
    ins = [xn.clone() for _ in range(G)]
    outs = [torch.zeros_like(xn) for _ in range(G)]
    run_virtual(shards, ins, outs)
    got = assemble_owned(shards, outs)
    ref = O.gather_scatter(e, n, x)
    vp = L.vertex_perm.cpu().numpy()
    ref_new = np.empty_like(ref)
    ref_new[vp] = ref
    assert np.array_equal(got.astype(np.float64), ref_new[:plan.touched])


def test_set_hub_split_rejects_below_minus_one():
    from paper_1605_02043_b200 import epg
    c = epg.Context(0)
    with pytest.raises(epg.EpgError) as ex:
        c.set_hub_split(-2)
    assert ex.value.status == epg.ERR_INPUT


@pytest.mark.parametrize("rows,edges", [(2048, 1024), (1536, 1024), (1024, 512), (128, 256), (64, 32)])
def test_exec_limits_rmat_exact(rmat14, rows, edges):
    """Execution-split caps (epg_set_exec_limits): wide caps run one-float rows with 8 rows
    per thread, narrow caps cut EP partitions into many ranges; all bit-exact."""
    from paper_1605_02043_b200 import epg
    n, e, P, part = rmat14
    x = S.int_vector(1613, n, 0, 7)
    ctx = _ctx(-1)
    ctx.set_exec_limits(rows, edges)
    got, plan = _scalar(ctx, epg.KERNEL_GATHER_SCATTER, e, n, part, O.num_parts(len(e), P), x)
    assert np.array_equal(got.astype(np.float64), O.gather_scatter(e, n, x))
    assert plan.k_exec >= plan.k
    if rows <= 128:
        assert plan.k_exec > 2 * plan.k


def test_exec_limits_wide_rows_cfd_falls_back(small_mesh):
    """cfd rows above 1024 do not fit the occupancy kernel: variant 3 refuses, variant 0
    runs another kernel, and the result still matches the oracle."""
    from paper_1605_02043_b200 import epg
    M = small_mesh
    P = 4096
    part = O.partition(M.edges, M.n, P)
    k = O.num_parts(M.m, P)
    U = S.cfd_state(M.n)
    dt = S.cfd_dt(M.volume).astype(np.float32)
    ref, _ = O.cfd_step(M.edges, M.n, M.normals, U, dt)
    for variant in (3, 0):
        ctx = _ctx(-1, variant)
        ctx.set_exec_limits(2048, 1024)
        L, plan = ctx.remap(dev(M.edges), M.n, dev(part), k)
        Un = ctx.permute_rows(dev(U), L.vertex_perm, epg.PERM_SCATTER)
        nrm = ctx.permute_rows(dev(M.normals), L.edge_perm, epg.PERM_GATHER)
        dtn = ctx.permute_rows(dev(dt), L.vertex_perm, epg.PERM_SCATTER)
        out = torch.empty_like(Un)
        try:
            ctx.run(plan, epg.KERNEL_CFD_FLUX, Un, out, nrm, dtn)
        except epg.EpgError as ex:                # an execution partition has > 1024 rows
            assert variant == 3 and ex.status == epg.ERR_INFEASIBLE
            continue
        got = ctx.permute_rows(out, L.vertex_perm, epg.PERM_GATHER).cpu().numpy()
        assert normwise_err(got, ref).max() <= TOL


def test_set_exec_limits_rejects_out_of_range():
    from paper_1605_02043_b200 import epg
    c = epg.Context(0)
    for r, e in ((63, 1024), (4096, 1024), (704, 31), (704, 2048), (-2, 1024)):
        with pytest.raises(epg.EpgError) as ex:
            c.set_exec_limits(r, e)
        assert ex.value.status == epg.ERR_INPUT
    c.set_exec_limits(-1, -1)

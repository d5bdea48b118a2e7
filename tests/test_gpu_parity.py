"""GPU parity: the CUDA path through the C ABI against the CPU oracle (oracle/).

Integer outputs (partition maps, load counts, remap permutations, halo sets, slots,
integer-valued functors) must be bit-exact; fp32 state within the normwise relative
tolerance of SURVEY Z14 / DESIGN.md: per component c,
max_v |x_gpu - x_ref| / max_v |x_ref| <= 1e-5 (north_star's "<= 1e-5 relative")."""
import numpy as np
import pytest
import torch

import oracle as O
import synth as S
from conftest import golden

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module", params=[0, 1, 2, 3], ids=["auto", "per_partition", "pipelined", "occupancy"])
def ctx(request):
    """Every staged-kernel variant: 0 automatic, 1 one CTA per partition with plain loads,
    2 persistent TMA-pipelined, 3 TMA-staged with several CTAs per SM."""
    from paper_1605_02043_b200 import epg
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    c = epg.Context(0)
    c.set_variant(request.param)
    return c


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def normwise_err(got, ref):
    got = np.asarray(got, np.float64).reshape(ref.shape[0], -1)
    ref = np.asarray(ref, np.float64).reshape(ref.shape[0], -1)
    return (np.abs(got - ref).max(axis=0) / np.maximum(np.abs(ref).max(axis=0), 1e-300))


# ---------------------------------------------------------------------------- cost (a3)
def _check_cost(ctx, edges, n, part, k):
    rep, pp = ctx.load_count(dev(edges), n, dev(part), k, per_part=True)
    r = O.cost(edges, n, part, k)
    assert (rep.k, rep.load_count, rep.touched, rep.cut_cost, rep.max_size, rep.min_size) == \
        (r.k, r.load_count, r.touched, r.cut_cost, r.max_size, r.min_size)
    assert np.array_equal(pp.cpu().numpy(), r.per_part)
    return rep


def test_cost_fig_mot(ctx):
    g = golden("fig_mot.json")
    for topo in g["topologies"].values():
        e = np.array(topo, np.int32)
        assert _check_cost(ctx, e, 6, np.array(g["schedule_a"], np.int32), 2).load_count == 9
        assert _check_cost(ctx, e, 6, np.array(g["schedule_b"], np.int32), 2).load_count == 7


@pytest.mark.parametrize("seed", range(12))
def test_cost_random(ctx, seed):
    rng = np.random.default_rng(2000 + seed)
    m, n = int(rng.integers(1, 5000)), int(rng.integers(1, 3000))
    n, e = S.random_multigraph(seed, m, n)
    k = int(rng.integers(1, 40))
    _check_cost(ctx, e, n, rng.integers(0, k, m).astype(np.int32), k)   # includes > 4096-edge partitions


@pytest.mark.parametrize("P", [256, 1024, 4096])
def test_cost_mesh(ctx, mesh_c1, P):
    M = mesh_c1
    k = O.num_parts(M.m, P)
    _check_cost(ctx, M.edges, M.n, O.default_partition(M.m, P), k)
    _check_cost(ctx, M.edges, M.n, O.partition(M.edges, M.n, P), k)


def test_default_partition(ctx):
    for m, P in [(1, 1), (7, 3), (190245, 1024), (458168, 256), (10000, 4096)]:
        assert np.array_equal(ctx.default_partition(m, P).cpu().numpy(), O.default_partition(m, P))


# ------------------------------------------------------------------------ partition (a2)
def test_partition_host_and_device_edges(ctx, mesh_c1):
    M = mesh_c1
    ref = O.partition(M.edges, M.n, 1024)
    r = O.cost(M.edges, M.n, ref, O.num_parts(M.m, 1024))
    part, rep = ctx.partition(dev(M.edges), M.n, 1024)
    assert np.array_equal(part.cpu().numpy(), ref)
    assert (rep.load_count, rep.cut_cost, rep.touched) == (r.load_count, r.cut_cost, r.touched)
    part_h, rep_h = ctx.partition(torch.from_numpy(M.edges), M.n, 1024)
    assert part_h.device.type == "cpu" and np.array_equal(part_h.numpy(), ref)
    assert rep_h == rep


# ---------------------------------------------------------------------------- remap (a4)
def _check_remap(ctx, edges, n, part, k, key=None):
    L, plan = ctx.remap(dev(edges), n, dev(part), k, order_key=None if key is None else dev(key))
    ref = O.remap(edges, n, part, k, key)
    for name in ("edge_perm", "part_edge_begin", "vertex_perm", "part_vertex_begin", "halo_begin", "halo_ids"):
        got = getattr(L, name).cpu().numpy()
        assert np.array_equal(got, getattr(ref, name)), name
    assert np.array_equal(L.slots.cpu().numpy(), ref.slots)
    r = O.cost(edges, n, part, k)
    assert plan.touched == r.touched and plan.cut_cost == r.cut_cost
    return L, plan


def test_remap_fixtures(ctx):
    g = golden("two_triangle.json")
    L, _ = _check_remap(ctx, np.array(g["edges"], np.int32), 6, np.array(g["optimal_partition"], np.int32), 2)
    assert L.part_vertex_begin.cpu().tolist() == g["optimal_block_begin"]
    g = golden("fig_mot.json")
    e = np.array(g["topologies"]["star_plus_triangle"], np.int32)
    _check_remap(ctx, e, 6, np.array(g["schedule_a"], np.int32), 2)
    _check_remap(ctx, e, 6, np.array(g["schedule_b"], np.int32), 2)


@pytest.mark.parametrize("seed", range(10))
def test_remap_random(ctx, seed):
    rng = np.random.default_rng(3000 + seed)
    m, n = int(rng.integers(1, 6000)), int(rng.integers(1, 3000))
    n, e = S.random_multigraph(seed, m, n)
    P = int(rng.choice([1, 7, 256, 1000, 4096]))
    k = O.num_parts(m, P)
    part = O.default_partition(m, P) if seed % 2 else O.partition(e, n, P)
    _check_remap(ctx, e, n, part, k)


@pytest.mark.parametrize("P", [256, 1024, 4096])
def test_remap_mesh(ctx, mesh_c1, P):
    M = mesh_c1
    k = O.num_parts(M.m, P)
    _check_remap(ctx, M.edges, M.n, O.partition(M.edges, M.n, P), k)
    _check_remap(ctx, M.edges, M.n, O.default_partition(M.m, P), k)


@pytest.mark.parametrize("seed", range(6))
def test_remap_keyed_random(ctx, seed):
    """epg_remap_keyed (reading Z22): arbitrary keys with ties, bit-exact vs orc_remap_keyed."""
    rng = np.random.default_rng(3100 + seed)
    m, n = int(rng.integers(1, 6000)), int(rng.integers(1, 3000))
    n, e = S.random_multigraph(40 + seed, m, n)
    P = int(rng.choice([7, 256, 1000, 4096]))
    k = O.num_parts(m, P)
    part = O.default_partition(m, P) if seed % 2 else O.partition(e, n, P)
    key = rng.integers(0, 50, m).astype(np.int32)
    _check_remap(ctx, e, n, part, k, key)


@pytest.mark.parametrize("P", [256, 1024, 4096])
def test_remap_growth_order_mesh(ctx, mesh_c1, P):
    """The growth-ranked layout of the EPG-2 map (what the bench runs), bit-exact; P = 4096
    also exercises the execution split (pieces of a growth-ordered partition)."""
    M = mesh_c1
    k = O.num_parts(M.m, P)
    part, rank = O.partition(M.edges, M.n, P, method=2, ranked=True)
    _check_remap(ctx, M.edges, M.n, part, k, rank)
    U, dt = _cfd_inputs(M)
    from paper_1605_02043_b200 import epg
    L, plan = ctx.remap(dev(M.edges), M.n, dev(part), k, order_key=dev(rank))
    Un = ctx.permute_rows(dev(U), L.vertex_perm, epg.PERM_SCATTER)
    nrm = ctx.permute_rows(dev(M.normals), L.edge_perm, epg.PERM_GATHER)
    dtn = ctx.permute_rows(dev(dt), L.vertex_perm, epg.PERM_SCATTER)
    out = torch.empty_like(Un)
    ctx.run(plan, epg.KERNEL_CFD_FLUX, Un, out, nrm, dtn, 1)
    got = ctx.permute_rows(out, L.vertex_perm, epg.PERM_GATHER).cpu().numpy()
    ref, _ = O.cfd_step(M.edges, M.n, M.normals, U, dt)
    assert normwise_err(got, ref).max() <= TOL


def test_remap_rejects_oversized_partition(ctx):
    from paper_1605_02043_b200 import epg
    n, e = S.random_multigraph(1, 5000, 100)
    with pytest.raises(epg.EpgError) as ex:
        ctx.remap(dev(e), n, torch.zeros(5000, dtype=torch.int32, device="cuda"), 1)
    assert ex.value.status == epg.ERR_INFEASIBLE


def test_errors(ctx):
    from paper_1605_02043_b200 import epg
    e = dev(np.array([[0, 1], [1, 9]], np.int32))
    with pytest.raises(epg.EpgError) as ex:
        ctx.load_count(e, 3, dev(np.zeros(2, np.int32)), 1)
    assert ex.value.status == epg.ERR_INPUT and "edge 1" in ex.value.message
    e = dev(np.array([[0, 1], [1, 2]], np.int32))
    with pytest.raises(epg.EpgError) as ex:
        ctx.load_count(e, 3, dev(np.array([0, 3], np.int32)), 2)
    assert ex.value.status == epg.ERR_INPUT
    with pytest.raises(epg.EpgError) as ex:
        ctx.remap(e, 3, dev(np.array([0, 1], np.int32)), 2, halo_cap=0)   # C = 1
    assert ex.value.status == epg.ERR_INPUT


# ------------------------------------------------------------------------- run (a5-a7)
def _cfd_inputs(M, dt_scale=1.0, seed=1606):
    U = S.cfd_state(M.n, seed)
    dt = (S.cfd_dt(M.volume) * dt_scale).astype(np.float32)
    return U, dt


def _run_cfd(ctx, M, part, k, U, dt, steps=1):
    from paper_1605_02043_b200 import epg
    E = dev(M.edges)
    L, plan = ctx.remap(E, M.n, dev(part), k)
    Un = ctx.permute_rows(dev(U), L.vertex_perm, epg.PERM_SCATTER)
    nrm = ctx.permute_rows(dev(M.normals), L.edge_perm, epg.PERM_GATHER)
    dtn = ctx.permute_rows(dev(dt), L.vertex_perm, epg.PERM_SCATTER)
    out = torch.empty_like(Un)
    res = ctx.run(plan, epg.KERNEL_CFD_FLUX, Un, out, nrm, dtn, steps=steps)
    return ctx.permute_rows(res, L.vertex_perm, epg.PERM_GATHER).cpu().numpy()


@pytest.mark.parametrize("sched", ["ep", "default"])
@pytest.mark.parametrize("P", [256, 1024, 2048])
def test_cfd_step_small_mesh(ctx, small_mesh, sched, P):
    M = small_mesh
    k = O.num_parts(M.m, P)
    part = O.partition(M.edges, M.n, P) if sched == "ep" else O.default_partition(M.m, P)
    U, dt = _cfd_inputs(M)
    got = _run_cfd(ctx, M, part, k, U, dt)
    ref, F = O.cfd_step(M.edges, M.n, M.normals, U, dt)
    assert np.abs(dt[:, None] * F).max() / np.abs(U).max() > 1e-3        # update is not vacuous (Z14)
    assert normwise_err(got, ref).max() <= TOL


def test_cfd_step_flux_dominated(ctx, small_mesh):
    """dt x1000: the result is dominated by dt*F, so the tolerance bounds the flux error."""
    M = small_mesh
    U, dt = _cfd_inputs(M, dt_scale=1000.0)
    part = O.partition(M.edges, M.n, 1024)
    got = _run_cfd(ctx, M, part, O.num_parts(M.m, 1024), U, dt)
    ref, F = O.cfd_step(M.edges, M.n, M.normals, U, dt)
    assert normwise_err(got, ref).max() <= TOL


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_cfd_step_full_size(ctx, name):
    """BASELINE configs C1/C2 at full size, P = 1024, every element compared."""
    M = S.config_mesh(name)
    k = O.num_parts(M.m, 1024)
    part, rep = ctx.partition(dev(M.edges), M.n, 1024)
    assert np.array_equal(part.cpu().numpy(), O.partition(M.edges, M.n, 1024))
    U, dt = _cfd_inputs(M)
    got = _run_cfd(ctx, M, part.cpu().numpy(), k, U, dt)
    ref, _ = O.cfd_step(M.edges, M.n, M.normals, U, dt)
    assert normwise_err(got, ref).max() <= TOL


def test_cfd_multi_step_and_determinism(ctx, small_mesh):
    """steps=2 equals two single steps bit for bit; each step is within tolerance of the
    oracle applied to the GPU's previous fp32 state (O8: one step at a time)."""
    M = small_mesh
    P = 512
    k = O.num_parts(M.m, P)
    part = O.partition(M.edges, M.n, P)
    U, dt = _cfd_inputs(M)
    s1 = _run_cfd(ctx, M, part, k, U, dt, steps=1)
    s1b = _run_cfd(ctx, M, part, k, U, dt, steps=1)
    assert np.array_equal(s1, s1b)
    s2 = _run_cfd(ctx, M, part, k, s1, dt, steps=1)
    s2_direct = _run_cfd(ctx, M, part, k, U, dt, steps=2)
    assert np.array_equal(s2, s2_direct)
    ref2, _ = O.cfd_step(M.edges, M.n, M.normals, s1, dt)
    assert normwise_err(s2, ref2).max() <= TOL


def test_occupancy_kernel_at_bench_config(ctx):
    """The bench configuration (C2, P = 1024) runs the occupancy TMA kernel (variant 3,
    which refuses to fall back to another variant) and matches the oracle at full size."""
    from paper_1605_02043_b200 import epg
    M = S.config_mesh("c2")
    k = O.num_parts(M.m, 1024)
    c2 = epg.Context(0)
    c2.set_variant(3)
    U, dt = _cfd_inputs(M)
    got = _run_cfd(c2, M, O.partition(M.edges, M.n, 1024), k, U, dt)
    ref, _ = O.cfd_step(M.edges, M.n, M.normals, U, dt)
    assert normwise_err(got, ref).max() <= TOL


def test_cfd_naive(ctx, small_mesh):
    from paper_1605_02043_b200 import epg
    M = small_mesh
    U, dt = _cfd_inputs(M)
    out = torch.empty((M.n, 5), dtype=torch.float32, device="cuda")
    ctx.run_naive(epg.KERNEL_CFD_FLUX, dev(M.edges), M.n, dev(U), out, dev(M.normals), dev(dt))
    ref, _ = O.cfd_step(M.edges, M.n, M.normals, U, dt)
    assert normwise_err(out.cpu().numpy(), ref).max() <= TOL


def test_cfd_hardware_cache_variant(ctx, small_mesh):
    """EP order + cpack layout through the unstaged kernel == the oracle."""
    from paper_1605_02043_b200 import epg
    M = small_mesh
    k = O.num_parts(M.m, 512)
    E = dev(M.edges)
    L, plan = ctx.remap(E, M.n, dev(O.partition(M.edges, M.n, 512)), k)
    Ex = ctx.remapped_edges(E, L)
    ref_lay = O.remap(M.edges, M.n, O.partition(M.edges, M.n, 512), k)
    assert np.array_equal(Ex.cpu().numpy(), ref_lay.vertex_perm[M.edges[ref_lay.edge_perm]])
    U, dt = _cfd_inputs(M)
    Un = ctx.permute_rows(dev(U), L.vertex_perm, epg.PERM_SCATTER)
    nrm = ctx.permute_rows(dev(M.normals), L.edge_perm, epg.PERM_GATHER)
    dtn = ctx.permute_rows(dev(dt), L.vertex_perm, epg.PERM_SCATTER)
    out = torch.empty_like(Un)
    ctx.run_naive(epg.KERNEL_CFD_FLUX, Ex, M.n, Un, out, nrm, dtn)
    got = ctx.permute_rows(out, L.vertex_perm, epg.PERM_GATHER).cpu().numpy()
    ref, _ = O.cfd_step(M.edges, M.n, M.normals, U, dt)
    assert normwise_err(got, ref).max() <= TOL


def test_cfd_untouched_vertices(ctx):
    """Isolated vertices (degree 0) keep their state (O8)."""
    M = S.kuhn_mesh(nbox=5, n_keep=700)
    n = M.n + 37
    edges = M.edges.copy()
    U = S.cfd_state(n)
    dt = np.full(n, 50.0, np.float32)

    class G:  # mesh with extra isolated vertices
        pass
    G.n, G.m, G.edges, G.normals = n, M.m, edges, M.normals
    part = O.partition(edges, n, 128)
    got = _run_cfd(ctx, G, part, O.num_parts(M.m, 128), U, dt)
    ref, _ = O.cfd_step(edges, n, M.normals, U, dt)
    assert np.array_equal(got[M.n:], U[M.n:])
    assert normwise_err(got, ref).max() <= TOL


def _run_scalar(ctx, kernel, edges, n, part, k, x, w):
    from paper_1605_02043_b200 import epg
    E = dev(edges)
    L, plan = ctx.remap(E, n, dev(part), k)
    xn = ctx.permute_rows(dev(x), L.vertex_perm, epg.PERM_SCATTER)
    wn = None if w is None else ctx.permute_rows(dev(w), L.edge_perm, epg.PERM_GATHER)
    out = torch.empty_like(xn)
    ctx.run(plan, kernel, xn, out, wn)
    return ctx.permute_rows(out, L.vertex_perm, epg.PERM_GATHER).cpu().numpy()


@pytest.mark.parametrize("seed", range(4))
def test_gather_scatter_integer_exact(ctx, seed):
    from paper_1605_02043_b200 import epg
    n, e = S.random_multigraph(seed, 20000, 3000)
    x = S.int_vector(seed, n, 0, 7)
    P = [64, 256, 1024, 4096][seed]
    part = O.partition(e, n, P)
    got = _run_scalar(ctx, epg.KERNEL_GATHER_SCATTER, e, n, part, O.num_parts(e.shape[0], P), x, None)
    assert np.array_equal(got.astype(np.float64), O.gather_scatter(e, n, x))
    xn = np.ones(n, np.float32)
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    ctx.run_naive(epg.KERNEL_GATHER_SCATTER, dev(e), n, dev(xn), out)
    assert np.array_equal(out.cpu().numpy(), np.bincount(e.ravel(), minlength=n).astype(np.float32))


def test_spmv_stencil_integer_exact(ctx):
    from paper_1605_02043_b200 import epg
    g = 60
    rows, cols, vals = [], [], []
    for i in range(g):
        for j in range(g):
            for di, dj, a in ((0, 0, 4.0), (-1, 0, -1.0), (1, 0, -1.0), (0, -1, -1.0), (0, 1, -1.0)):
                if 0 <= i + di < g and 0 <= j + dj < g:
                    rows.append(i * g + j); cols.append((i + di) * g + j + dj); vals.append(a)
    N = g * g
    edges = np.stack([np.array(cols), N + np.array(rows)], axis=1).astype(np.int32)
    w = np.array(vals, np.float32)
    x = np.concatenate([S.int_vector(5, N, -8, 8), np.zeros(N, np.float32)])
    ref = O.spmv(edges, 2 * N, w, x)
    for part, P in ((O.partition(edges, 2 * N, 512), 512), (O.default_partition(edges.shape[0], 1024), 1024)):
        got = _run_scalar(ctx, epg.KERNEL_SPMV, edges, 2 * N, part, O.num_parts(edges.shape[0], P), x, w)
        assert np.array_equal(got.astype(np.float64), ref)
    out = torch.empty(2 * N, dtype=torch.float32, device="cuda")
    ctx.run_naive(epg.KERNEL_SPMV, dev(edges), 2 * N, dev(x), out, dev(w))
    assert np.array_equal(out.cpu().numpy().astype(np.float64), ref)


def test_single_edge_and_p1(ctx):
    from paper_1605_02043_b200 import epg
    e = np.array([[0, 1]], np.int32)
    x = np.array([3, 5], np.float32)
    got = _run_scalar(ctx, epg.KERNEL_GATHER_SCATTER, e, 2, np.zeros(1, np.int32), 1, x, None)
    assert got.tolist() == [5.0, 3.0]
    n, e = S.random_multigraph(4, 300, 50)    # P = 1: every task its own partition
    x = S.int_vector(4, n, 0, 7)
    got = _run_scalar(ctx, epg.KERNEL_GATHER_SCATTER, e, n, O.partition(e, n, 1), 300, x, None)
    assert np.array_equal(got.astype(np.float64), O.gather_scatter(e, n, x))


@pytest.mark.parametrize("P", [512, 1024])
def test_rmat_gather_scatter_exact(ctx, P):
    """C4's shape at scale 14 (hubs, self-loops, duplicates): EP partition through the
    library, staged kernel, integer-valued x -> bit-exact vs the oracle."""
    from paper_1605_02043_b200 import epg
    n, e = S.rmat(14)
    x = S.int_vector(1608, n, 0, 7)
    k = O.num_parts(e.shape[0], P)
    E = dev(e)
    part, rep = ctx.partition(E, n, P)
    assert np.array_equal(part.cpu().numpy(), O.partition(e, n, P))
    got = _run_scalar(ctx, epg.KERNEL_GATHER_SCATTER, e, n, part.cpu().numpy(), k, x, None)
    assert np.array_equal(got.astype(np.float64), O.gather_scatter(e, n, x))


def test_stencil_spmv_c5_shape_exact(ctx):
    """C5's shape (2D 5-point Laplacian, bipartite COO in row-major order) at g = 300."""
    from paper_1605_02043_b200 import epg
    n, e, w = S.stencil2d_spmv(300)
    N = n // 2
    x = np.concatenate([S.int_vector(1609, N, -8, 8), np.zeros(N, np.float32)])
    P = 1024
    k = O.num_parts(e.shape[0], P)
    part, _ = ctx.partition(dev(e), n, P)
    got = _run_scalar(ctx, epg.KERNEL_SPMV, e, n, part.cpu().numpy(), k, x, w)
    assert np.array_equal(got.astype(np.float64), O.spmv(e, n, w, x))

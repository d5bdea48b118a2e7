"""One small run of the staged edge kernel + finalise for compute-sanitizer.

    compute-sanitizer --tool racecheck python tools/sanitize.py c1_single

Scenarios: the launch shapes the bench uses, at sizes the sanitizers finish in minutes.
  c1_single    C1 mesh, P = 1024, EPG-2 map: one wave, early halo gather, early PDL trigger
  c1_multiwave C1 mesh, P = 32: ~6,000 execution partitions, next-wave L2 prefetch, late PDL
  default_map  C1 mesh, P = 1024, default (contiguous) map: halo-heavy partitions, late gather
  hub          R-MAT scale 14, gather-scatter, hub split on (red.global.add accumulators)
  spmv         2D 5-point stencil SpMV (bipartite graph), P = 1024
  wide         C1 mesh, P = 1100: the 288-thread (9-warp) instance, single wave
  sharded      C1 mesh, P = 1024, in-process group of 4: interior / boundary launches, exchange
Every plan carries the bank-conflict placement (place.cpp) unless EPG_PLACE=0; the hub
scenario's variable-length incidence lists take the segmented-scan reduce.
Each checks its result against the fp64 oracle, so a run that the sanitizer perturbs
into a wrong answer fails loudly too.
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("EPG_GRAPHS", "0")   # individual launches (the graph replays the same kernels)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import synth as S  # noqa: E402
from paper_1605_02043_b200 import epg  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def cfd(M, P, default_map=False):
    ctx = epg.Context(0)
    ctx.set_partition_method(2)
    if P > 1024:
        ctx.set_exec_limits(1152, 1152)
    k = epg.num_parts(M.m, P)
    E = dev(M.edges)
    part = ctx.default_partition(M.m, P) if default_map else ctx.partition(E, M.n, P)[0]
    L, plan = ctx.remap(E, M.n, part, k)
    U, dt = S.cfd_state(M.n), S.cfd_dt(M.volume)
    Un = ctx.permute_rows(dev(U), L.vertex_perm, epg.PERM_SCATTER)
    nrm = ctx.permute_rows(dev(M.normals), L.edge_perm, epg.PERM_GATHER)
    dtn = ctx.permute_rows(dev(dt), L.vertex_perm, epg.PERM_SCATTER)
    out = torch.empty_like(Un)
    ctx.run(plan, epg.KERNEL_CFD_FLUX, Un, out, nrm, dtn, 1)
    got = ctx.permute_rows(out, L.vertex_perm, epg.PERM_GATHER).cpu().numpy().astype(np.float64)
    ref, _ = O.cfd_step(M.edges, M.n, M.normals, U, dt)
    err = (np.abs(got - ref).max(axis=0) / np.abs(ref).max(axis=0)).max()
    print(f"cfd m={M.m} P={P} k_exec={plan.k_exec} err={err:.2e}")
    assert err <= 1e-5


def hub():
    n, e = S.rmat(14)
    P = 512
    ctx = epg.Context(0)
    ctx.set_variant(3)
    ctx.set_hub_split(7)
    part = O.partition(e, n, P)
    L, plan = ctx.remap(dev(e), n, dev(part), O.num_parts(len(e), P))
    x = S.int_vector(1608, n, 0, 7)
    xn = ctx.permute_rows(dev(x), L.vertex_perm, epg.PERM_SCATTER)
    out = torch.empty_like(xn)
    ctx.run(plan, epg.KERNEL_GATHER_SCATTER, xn, out, None, None, 1)
    got = ctx.permute_rows(out, L.vertex_perm, epg.PERM_GATHER).cpu().numpy().astype(np.float64)
    print(f"hub m={len(e)} hubs={plan.hubs} k_exec={plan.k_exec}")
    assert np.array_equal(got, O.gather_scatter(e, n, x))


def spmv():
    n, e, w = S.stencil2d_spmv(300)
    N = n // 2
    P = 1024
    ctx = epg.Context(0)
    ctx.set_partition_method(2)
    part, _ = ctx.partition(dev(e), n, P)
    L, plan = ctx.remap(dev(e), n, part, epg.num_parts(len(e), P))
    x = np.concatenate([S.int_vector(1609, N, -8, 8), np.zeros(N, np.float32)])
    xn = ctx.permute_rows(dev(x), L.vertex_perm, epg.PERM_SCATTER)
    wn = ctx.permute_rows(dev(w), L.edge_perm, epg.PERM_GATHER)
    out = torch.empty_like(xn)
    ctx.run(plan, epg.KERNEL_SPMV, xn, out, wn, None, 1)
    got = ctx.permute_rows(out, L.vertex_perm, epg.PERM_GATHER).cpu().numpy().astype(np.float64)
    print(f"spmv m={len(e)} k_exec={plan.k_exec}")
    assert np.array_equal(got, O.spmv(e, n, w, x))


def sharded():
    M = S.config_mesh("c1")
    G, P = 4, 1024
    ctxs = [epg.Context(0) for _ in range(G)]
    k = epg.num_parts(M.m, P)
    E = dev(M.edges)
    part, rank, _ = ctxs[0].partition_rb(E, M.n, P, G, 8, ranked=True)
    U, dt = S.cfd_state(M.n), S.cfd_dt(M.volume)
    plans, states = [], []
    for c in ctxs:
        L, plan = c.remap(E, M.n, part, k, order_key=rank)
        Un = c.permute_rows(dev(U), L.vertex_perm, epg.PERM_SCATTER)
        nrm = c.permute_rows(dev(M.normals), L.edge_perm, epg.PERM_GATHER)
        dtn = c.permute_rows(dev(dt), L.vertex_perm, epg.PERM_SCATTER)
        plans.append(plan)
        states.append((Un, torch.empty_like(Un), nrm, dtn, L))
    epg.comm_init_local(ctxs)
    epg.run_sharded_group(ctxs, plans, epg.KERNEL_CFD_FLUX, [s[:4] for s in states])
    torch.cuda.synchronize()
    ref, _ = O.cfd_step(M.edges, M.n, M.normals, U, dt)
    vp = states[0][4].vertex_perm.cpu().numpy()
    ref_l = np.empty_like(ref)
    ref_l[vp] = ref                                   # the oracle's rows in the plan layout
    err = 0.0
    for g in range(G):   # each member's own (authoritative) rows
        out = states[g][1]
        r = ctxs[g].shard_ranges(plans[g], G, g)
        lo, hi = r["vertex_first"], r["vertex_first"] + r["vertex_count"]
        got = out[lo:hi].cpu().numpy().astype(np.float64)
        err = max(err, (np.abs(got - ref_l[lo:hi]).max(axis=0) / np.abs(ref).max(axis=0)).max())
    print(f"sharded G={G} k={k} err={err:.2e}")
    assert err <= 1e-5


def main(which):
    if which == "c1_single":
        cfd(S.config_mesh("c1"), 1024)
    elif which == "c1_multiwave":
        cfd(S.config_mesh("c1"), 32)
    elif which == "default_map":
        cfd(S.config_mesh("c1"), 1024, default_map=True)
    elif which == "hub":
        hub()
    elif which == "spmv":
        spmv()
    elif which == "wide":
        cfd(S.config_mesh("c1"), 1100)
    elif which == "sharded":
        sharded()
    else:
        raise SystemExit(f"unknown scenario {which}")
    torch.cuda.synchronize()
    print(f"{which}: ok")


if __name__ == "__main__":
    main(sys.argv[1])

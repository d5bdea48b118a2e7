"""The sharded path with the real kernels: G virtual shards on one GPU, each
with its own full-size state whose foreign rows start stale, exchanging through tensor
copies (the NCCL transfers of a multi-GPU run carry the same buffers)."""
import numpy as np
import pytest
import torch

import oracle as O
import synth as S

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("P,method", [(1024, 1), (2048, 1), (1024, 2)])
def test_virtual_shards_cfd(mesh_c1, G, P, method):
    from paper_1605_02043_b200 import epg
    from paper_1605_02043_b200.shard import Shard, run_virtual, assemble_owned
    M = mesh_c1
    k = O.num_parts(M.m, P)
    ctx = epg.Context(0)
    ctx.set_partition_method(method)
    E = torch.from_numpy(M.edges).cuda()
    part, _ = ctx.partition(E, M.n, P, shards=G)
    assert np.array_equal(part.cpu().numpy(), O.partition(M.edges, M.n, P, G, method=method))   # hierarchical EPG
    L, plan = ctx.remap(E, M.n, part, k)
    U, dt = S.cfd_state(M.n), S.cfd_dt(M.volume)
    Un = ctx.permute_rows(torch.from_numpy(U).cuda(), L.vertex_perm, epg.PERM_SCATTER)
    nrm = ctx.permute_rows(torch.from_numpy(M.normals).cuda(), L.edge_perm, epg.PERM_GATHER)
    dtn = ctx.permute_rows(torch.from_numpy(dt).cuda(), L.vertex_perm, epg.PERM_SCATTER)
    shards = [Shard(ctx, plan, L, epg.KERNEL_CFD_FLUX, G, g) for g in range(G)]
    ins, outs = [], []
    for sh in shards:
        lo, hi = sh.owned()
        s = Un.clone()
        s[:lo] = 1e9                        # foreign rows stale: the pull must deliver them
        s[hi:plan.touched] = 1e9
        ins.append(s)
        outs.append(torch.zeros_like(Un))
    assert sum(v.numel() for sh in shards for v in sh.recv_ids.values()) > 0
    run_virtual(shards, ins, outs, nrm, dtn)
    got_new = assemble_owned(shards, outs)
    ref, _ = O.cfd_step(M.edges, M.n, M.normals, U, dt)
    vp = L.vertex_perm.cpu().numpy()
    ref_new = np.empty_like(ref)
    ref_new[vp] = ref
    err = np.abs(got_new - ref_new[:plan.touched]).max(axis=0) / np.abs(ref).max(axis=0)
    assert err.max() <= 1e-5
    # and against the single-GPU run of the same plan
    one = torch.empty_like(Un)
    ctx.run(plan, epg.KERNEL_CFD_FLUX, Un.clone(), one, nrm, dtn)
    d = np.abs(got_new - one[:plan.touched].cpu().numpy()).max() / np.abs(ref).max()
    assert d <= 1e-6


def test_virtual_shards_gather_scatter_exact():
    from paper_1605_02043_b200 import epg
    from paper_1605_02043_b200.shard import Shard, run_virtual, assemble_owned
    n, e = S.random_multigraph(9, 30000, 5000)
    x = S.int_vector(9, n, 0, 7)
    P, G = 512, 4
    k = O.num_parts(e.shape[0], P)
    ctx = epg.Context(0)
    E = torch.from_numpy(e).cuda()
    part, _ = ctx.partition(E, n, P, shards=G)
    L, plan = ctx.remap(E, n, part, k)
    xn = ctx.permute_rows(torch.from_numpy(x).cuda(), L.vertex_perm, epg.PERM_SCATTER)
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

"""GPU: epg_run_host, the end-to-end call from and to host memory (include/epg.h).

Several calls in flight (double-buffered staging, copy-in / compute / copy-out streams)
must each return exactly what the device-buffer path (permute_rows + epg_run + permute_rows)
returns for the same input, bit for bit, and the cfd step must stay within the Z14
tolerance of the fp64 oracle."""
import numpy as np
import pytest
import torch

import oracle as O
import synth as S

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _setup(M, P=256):
    from paper_1605_02043_b200 import epg
    ctx = epg.Context(0)
    k = O.num_parts(M.m, P)
    part, _ = ctx.partition(dev(M.edges), M.n, P)
    L, plan = ctx.remap(dev(M.edges), M.n, part, k)
    return ctx, L, plan


def _device_path(ctx, L, plan, kernel, U, pay, vc, steps):
    from paper_1605_02043_b200 import epg
    Un = ctx.permute_rows(dev(U), L.vertex_perm, epg.PERM_SCATTER)
    out = torch.empty_like(Un)
    res = ctx.run(plan, kernel, Un, out, pay, vc, steps) if steps else Un
    return ctx.permute_rows(res, L.vertex_perm, epg.PERM_GATHER).cpu().numpy()


@pytest.mark.parametrize("steps", [0, 1, 2])
def test_run_host_cfd_pipelined(steps):
    from paper_1605_02043_b200 import epg
    M = S.kuhn_mesh(nbox=12, n_keep=9000)
    ctx, L, plan = _setup(M)
    dt = S.cfd_dt(M.volume)
    nrm = ctx.permute_rows(dev(M.normals), L.edge_perm, epg.PERM_GATHER)
    dtn = ctx.permute_rows(dev(dt), L.vertex_perm, epg.PERM_SCATTER)
    inputs = [S.cfd_state(M.n, seed) for seed in (11, 12, 13, 14, 15)]
    hin = [torch.from_numpy(u).pin_memory() for u in inputs]
    hout = [torch.full_like(h, float("nan")).pin_memory() for h in hin]
    for a, b in zip(hin, hout):                    # five calls in flight, no sync in between
        ctx.run_host(plan, epg.KERNEL_CFD_FLUX, L.vertex_perm, a, b, nrm, dtn, steps)
    ctx.join()
    torch.cuda.current_stream().synchronize()
    for u, b in zip(inputs, hout):
        want = _device_path(ctx, L, plan, epg.KERNEL_CFD_FLUX, u, nrm, dtn, steps)
        assert np.array_equal(b.numpy(), want)
    if steps == 1:
        ref, _ = O.cfd_step(M.edges, M.n, M.normals, inputs[0], dt)
        err = np.abs(hout[0].numpy() - ref).max(axis=0) / np.abs(ref).max(axis=0)
        assert err.max() <= 1e-5


def test_run_host_gather_scatter_exact_and_errors():
    from paper_1605_02043_b200 import epg
    n, e = S.random_multigraph(3, 20000, 3000)
    P = 512
    ctx = epg.Context(0)
    k = O.num_parts(e.shape[0], P)
    part = O.partition(e, n, P)
    L, plan = ctx.remap(dev(e), n, dev(part), k)
    x = S.int_vector(3, n, 0, 7)
    hin = torch.from_numpy(x).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    ctx.run_host(plan, epg.KERNEL_GATHER_SCATTER, L.vertex_perm, hin, hout)
    ctx.join()
    torch.cuda.current_stream().synchronize()
    assert np.array_equal(hout.numpy().astype(np.float64), O.gather_scatter(e, n, x))
    with pytest.raises(epg.EpgError) as ex:                 # unknown kernel id
        ctx._check(epg.lib.epg_run_host(ctx.handle, plan.handle, 9, L.vertex_perm.data_ptr(), hin.data_ptr(),
                                        hout.data_ptr(), None, None, 1))
    assert ex.value.status == epg.ERR_INPUT
    with pytest.raises(ValueError):                         # device tensors are not host state
        ctx.run_host(plan, epg.KERNEL_GATHER_SCATTER, L.vertex_perm, hin.cuda(), hout)

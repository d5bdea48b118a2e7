"""Host-side cost of one epg_run call from Python (C2 plan, graph replay), and the device
time of back-to-back calls: is a per-step Python loop host-bound?"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth as S  # noqa: E402
from paper_1605_02043_b200 import epg  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    ctx = epg.Context(0, stream)
    ctx.set_partition_method(2)
    M = S.config_mesh("c2")
    E = torch.from_numpy(M.edges).cuda()
    part, rep = ctx.partition(E, M.n, 1024)
    L, plan = ctx.remap(E, M.n, part, epg.num_parts(M.m, 1024), halo_cap=rep.cut_cost)
    U = torch.from_numpy(S.cfd_state(M.n)).cuda()
    nrm = ctx.permute_rows(torch.from_numpy(M.normals).cuda(), L.edge_perm, epg.PERM_GATHER)
    dtn = ctx.permute_rows(torch.from_numpy(S.cfd_dt(M.volume)).cuda(), L.vertex_perm, epg.PERM_SCATTER)
    a = ctx.permute_rows(U, L.vertex_perm, epg.PERM_SCATTER)
    b = torch.empty_like(a)
    out = {}
    for i in range(20):
        ctx.run(plan, epg.KERNEL_CFD_FLUX, a, b, nrm, dtn, 1)
    torch.cuda.synchronize()
    N = 2000
    # host time per call, GPU kept busy by a long kernel first so nothing blocks
    big = torch.empty(1 << 28, device=dev)
    big.fill_(1.0)
    t0 = time.perf_counter()
    for i in range(N):
        ctx.run(plan, epg.KERNEL_CFD_FLUX, a, b, nrm, dtn, 1)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    out["host_us_per_epg_run_call"] = (t1 - t0) / N * 1e6
    # raw ctypes call without the Python wrapper
    st = epg._State(a.data_ptr(), b.data_ptr(), nrm.data_ptr(), dtn.data_ptr())
    import ctypes as C
    f = epg.lib.epg_run
    h, ph, ref = ctx.handle, plan.handle, C.byref(st)
    big.fill_(1.0)
    t0 = time.perf_counter()
    for i in range(N):
        f(h, ph, 1, ref, 1)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    out["host_us_per_raw_ctypes_call"] = (t1 - t0) / N * 1e6
    # device time per step, back to back
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    big.fill_(1.0)
    e0.record(stream)
    for i in range(N):
        f(h, ph, 1, ref, 1)
    e1.record(stream)
    torch.cuda.synchronize()
    out["device_us_per_step_back_to_back_calls"] = e0.elapsed_time(e1) * 1e3 / N
    e0.record(stream)
    ctx.run(plan, epg.KERNEL_CFD_FLUX, a, b, nrm, dtn, 200)
    e1.record(stream)
    torch.cuda.synchronize()
    out["device_us_per_step_one_call_200_steps"] = e0.elapsed_time(e1) * 1e3 / 200
    print(json.dumps(out, indent=1))


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def replicas():
    """Device time per step when consecutive steps run on R different plans (replicas)."""
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    ctx = epg.Context(0, stream)
    ctx.set_partition_method(2)
    M = S.config_mesh("c2")
    E = torch.from_numpy(M.edges).cuda()
    part, rep = ctx.partition(E, M.n, 1024)
    U = torch.from_numpy(S.cfd_state(M.n)).cuda()
    nrm0 = torch.from_numpy(M.normals).cuda()
    dt0 = torch.from_numpy(S.cfd_dt(M.volume)).cuda()
    reps = []
    for r in range(24):
        L, plan = ctx.remap(E, M.n, part, epg.num_parts(M.m, 1024), halo_cap=rep.cut_cost)
        nrm = ctx.permute_rows(nrm0, L.edge_perm, epg.PERM_GATHER)
        dtn = ctx.permute_rows(dt0, L.vertex_perm, epg.PERM_SCATTER)
        a = ctx.permute_rows(U, L.vertex_perm, epg.PERM_SCATTER)
        reps.append((plan, a, torch.empty_like(a), nrm, dtn))
    out = {}
    for R in (1, 2, 4, 8, 24):
        for i in range(2 * R):
            p, a, b, nrm, dtn = reps[i % R]
            ctx.run(p, epg.KERNEL_CFD_FLUX, a, b, nrm, dtn, 1)
        torch.cuda.synchronize()
        N = 480
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(N):
            p, a, b, nrm, dtn = reps[i % R]
            ctx.run(p, epg.KERNEL_CFD_FLUX, a, b, nrm, dtn, 1)
        e1.record(stream)
        torch.cuda.synchronize()
        out[f"R{R}_device_us_per_step"] = e0.elapsed_time(e1) * 1e3 / N
    print(json.dumps(out, indent=1))


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "replicas":
    replicas()

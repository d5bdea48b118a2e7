"""Measurement-floor experiment: what do two CUDA events around a step cost after an L2 flush?

Compares, on the C2 workload (EPG-2, P = 1024): an empty kernel and one epg_run step, each
timed with events after (a) a 512 MiB write flush, (b) the write flush followed by a 256 MiB
read pass that evicts the flush's dirty lines (our inputs are still not in L2), (c) no flush;
plus K steps in one epg_run call (steady state, L2 warm).
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth as S  # noqa: E402
from paper_1605_02043_b200 import epg  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    ctx = epg.Context(0, stream)
    ctx.set_partition_method(2)
    M = S.config_mesh("c2")
    P = 1024
    E = torch.from_numpy(M.edges).cuda()
    part, rep = ctx.partition(E, M.n, P)
    L, plan = ctx.remap(E, M.n, part, epg.num_parts(M.m, P), halo_cap=rep.cut_cost)
    U = torch.from_numpy(S.cfd_state(M.n)).cuda()
    nrm = ctx.permute_rows(torch.from_numpy(M.normals).cuda(), L.edge_perm, epg.PERM_GATHER)
    dtn = ctx.permute_rows(torch.from_numpy(S.cfd_dt(M.volume)).cuda(), L.vertex_perm, epg.PERM_SCATTER)
    bufs = [ctx.permute_rows(U, L.vertex_perm, epg.PERM_SCATTER), torch.empty_like(U)]
    wbuf = torch.empty(512 << 18, dtype=torch.float32, device=dev)
    rbuf = torch.ones(256 << 18, dtype=torch.float32, device=dev)
    sink = torch.empty(1, dtype=torch.float32, device=dev)
    tiny = torch.empty(1, dtype=torch.float32, device=dev)

    def flush_w():
        wbuf.fill_(1.0)

    def flush_wr():
        wbuf.fill_(1.0)
        torch.sum(rbuf, dim=0, out=sink)

    def none():
        pass

    def empty():
        tiny.fill_(0.0)

    def step(i):
        ctx.run(plan, epg.KERNEL_CFD_FLUX, bufs[i & 1], bufs[1 - (i & 1)], nrm, dtn, 1)

    def timed(flush, body, K=200):
        for i in range(5):
            flush(); body(i)
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for i in range(K):
            flush()
            evs[i][0].record(stream)
            body(i)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        t = [a.elapsed_time(b) * 1e3 for a, b in evs]
        return {"mean_us": float(np.mean(t)), "median_us": float(np.median(t)), "min_us": float(np.min(t))}

    out = {}
    for fname, f in (("write_flush", flush_w), ("write_then_read", flush_wr), ("no_flush", none)):
        out[fname] = {"empty_kernel": timed(f, lambda i: empty()), "c2_step": timed(f, step)}
    # steady state: K steps in one call (graph of K steps), L2 warm
    for K in (10, 100):
        a, b = bufs[0].clone(), bufs[1].clone()
        ctx.run(plan, epg.KERNEL_CFD_FLUX, a, b, nrm, dtn, K)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.run(plan, epg.KERNEL_CFD_FLUX, a, b, nrm, dtn, K)
        e1.record(stream)
        torch.cuda.synchronize()
        out[f"steady_{K}_steps_one_call_us_per_step"] = e0.elapsed_time(e1) * 1e3 / K
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

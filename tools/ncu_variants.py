"""Run one cfd time step of each schedule variant on a mesh, for ncu capture.

    ncu --metrics <...> -k regex:'k_edge|k_finalise|k_naive' python tools/ncu_variants.py --config c2

Variants, in launch order: EP staged with the EPG-2 map ("ep"; edge kernel + finalise), the
EPG-RB map ("rb", the bench's partitioner on C3),
EP staged with the EPG-1 map ("ep1"), default-map staged (same kernels), naive original
order (k_naive_edges + k_naive_update). `--reps R`
repeats the sequence (ncu -s can skip the first). Prints the per-variant kernel order.
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth as S  # noqa: E402
from paper_1605_02043_b200 import epg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--part-size", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--variants", default="ep,ep1,default,naive")
    a = ap.parse_args()
    if a.config in ("c4", "c5"):   # R-MAT gather-scatter / stencil SpMV: bench.py's workload
        import bench
        W = bench.Workload(a.config)
        M = argparse.Namespace(n=W.n, m=W.m, edges=W.edges, normals=W.payload)
        U, dt, KER = W.state, W.vconst, W.kernel
    else:
        M = S.config_mesh(a.config)
        U, dt, KER = S.cfd_state(M.n), S.cfd_dt(M.volume), epg.KERNEL_CFD_FLUX
    ctx = epg.Context(0)
    if a.config == "c4":
        ctx.set_exec_limits(1024, 1024)
    E = torch.from_numpy(M.edges).cuda()
    k = epg.num_parts(M.m, a.part_size)
    Ud = torch.from_numpy(U).cuda()
    runs = []
    for v in a.variants.split(","):
        if v in ("ep", "ep1", "default", "rb"):
            key = None
            if v == "default":
                part = ctx.default_partition(M.m, a.part_size)
            elif v == "rb":       # the bench's map and layout: EPG-RB, tasks in growth order (Z22)
                part, key, _ = ctx.partition_rb(E, M.n, a.part_size, 1, 4096 if a.config == "c4" else 512, ranked=True)
            else:
                ctx.set_partition_method(epg.PARTITION_EPG2 if v == "ep" else epg.PARTITION_EPG1)
                part = ctx.partition(E, M.n, a.part_size)[0]
            L, plan = ctx.remap(E, M.n, part, k, order_key=key)
            nrm = None if M.normals is None else ctx.permute_rows(torch.from_numpy(M.normals).cuda(), L.edge_perm,
                                                                   epg.PERM_GATHER)
            dtn = None if dt is None else ctx.permute_rows(torch.from_numpy(dt).cuda(), L.vertex_perm,
                                                           epg.PERM_SCATTER)
            b = [ctx.permute_rows(Ud, L.vertex_perm, epg.PERM_SCATTER), torch.empty_like(Ud)]
            runs.append((v, lambda plan=plan, b=b, nrm=nrm, dtn=dtn:
                         ctx.run(plan, KER, b[0], b[1], nrm, dtn, 1), plan))
        else:
            b = [Ud.clone(), torch.empty_like(Ud)]
            nrm0 = None if M.normals is None else torch.from_numpy(M.normals).cuda()
            dt0 = None if dt is None else torch.from_numpy(dt).cuda()
            runs.append((v, lambda b=b, nrm0=nrm0, dt0=dt0:
                         ctx.run_naive(KER, E, M.n, b[0], b[1], nrm0, dt0, 1), None))
    torch.cuda.synchronize()
    for r in range(a.reps):
        for name, fn, plan in runs:
            fn()
            torch.cuda.synchronize()
            if r == 0:
                extra = (f" k={plan.k} k_exec={plan.k_exec} touched={plan.touched} C={plan.cut_cost} "
                         f"C_exec={plan.cut_cost_exec} S={plan.shared}") if plan else ""
                print(f"variant {name}: m={M.m} n={M.n}{extra}", flush=True)


if __name__ == "__main__":
    main()

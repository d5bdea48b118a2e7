"""Per-phase %globaltimer trace of the staged edge kernel (development tool, GPU box).

Builds a -DEPG_TRACE copy of libepg.so (tools/_trace/libepg_trace.so), runs one L2-cold
cfd step of the bench workload and prints, per trace point of k_edge_occ, the
distribution over CTAs of (stamp - earliest CTA start) in microseconds.

    python tools/trace_phases.py [--config c2] [--part-size 1024] [--reps 3]
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tools", "_trace")


def build_trace_lib() -> str:
    sys.path.insert(0, os.path.join(ROOT, "paper_1605_02043_b200"))
    import build as b  # noqa: E402  (paper_1605_02043_b200/build.py, loaded by path)
    os.makedirs(OUT, exist_ok=True)
    lib = os.path.join(OUT, "libepg_trace.so")
    cmd = [b.nvcc(), "-O3", "-std=c++17", *b.ARCH, "-lineinfo", "-DEPG_TRACE", "-Xcompiler", "-fPIC", "-shared",
           *[os.path.join(b.CSRC, s) for s in b.SOURCES], "-o", lib]
    if not os.path.exists(lib) or any(os.path.getmtime(os.path.join(b.CSRC, s)) > os.path.getmtime(lib)
                                      for s in os.listdir(b.CSRC)):
        subprocess.check_call(cmd)
    return lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--part-size", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--variants", default="0")
    ap.add_argument("--rr", type=int, default=0,
                    help="R > 0: trace the last step of 2R round-robin steps over R replicas (bench.py's "
                         "headline mode: direct launches chained by PDL, inputs evicted) instead of one cold step")
    ap.add_argument("--chain", action="store_true",
                    help="with --rr: trace the finalise of the last step and the edge kernel launched after it "
                         "(times relative to the earliest finalise CTA start)")
    a = ap.parse_args()
    os.environ["EPG_LIB_PATH"] = build_trace_lib()
    sys.path.insert(0, ROOT)
    import ctypes as C

    import numpy as np
    import torch

    import synth as S
    from paper_1605_02043_b200 import epg

    epg.lib.epg_debug_trace.restype = C.c_int
    epg.lib.epg_debug_trace.argtypes = [C.c_void_p, C.c_int64]
    M = S.config_mesh(a.config)
    U, dt = S.cfd_state(M.n), S.cfd_dt(M.volume)
    ctx = epg.Context(0)
    E = torch.from_numpy(M.edges).cuda()
    k = epg.num_parts(M.m, a.part_size)
    part, rank, _ = ctx.partition_rb(E, M.n, a.part_size, ranked=True)   # the bench's map and order
    L, plan = ctx.remap(E, M.n, part, k, order_key=rank)
    nrm = ctx.permute_rows(torch.from_numpy(M.normals).cuda(), L.edge_perm, epg.PERM_GATHER)
    dtn = ctx.permute_rows(torch.from_numpy(dt).cuda(), L.vertex_perm, epg.PERM_SCATTER)
    Un = ctx.permute_rows(torch.from_numpy(U).cuda(), L.vertex_perm, epg.PERM_SCATTER)
    out = torch.empty_like(Un)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    npts, niters = 8, 16
    nblk = min(plan.k_exec, 1024)
    epg.lib.epg_debug_trace_clear.restype = C.c_int
    runs = [(v, rep) for v in map(int, a.variants.split(",")) for rep in range(a.reps)]
    reps = []
    if a.rr:
        for r in range(a.rr):
            Lr, pr = ctx.remap(E, M.n, part, k, order_key=rank)
            reps.append((pr, ctx.permute_rows(torch.from_numpy(U).cuda(), Lr.vertex_perm, epg.PERM_SCATTER),
                         ctx.permute_rows(torch.from_numpy(M.normals).cuda(), Lr.edge_perm, epg.PERM_GATHER),
                         ctx.permute_rows(torch.from_numpy(dt).cuda(), Lr.vertex_perm, epg.PERM_SCATTER)))
        reps = [(pr, u, torch.empty_like(u), nr, dd) for pr, u, nr, dd in reps]
    for v, rep in runs:
        ctx.set_variant(v)
        torch.cuda.synchronize()
        if a.rr:
            for i in range(2 * a.rr):              # warm: every replica twice
                pr, u, o, nr, dd = reps[i % a.rr]
                ctx.run(pr, epg.KERNEL_CFD_FLUX, u, o, nr, dd, 1)
            torch.cuda.synchronize()
            torch.cuda._sleep(2_000_000)
            for i in range(2 * a.rr):              # the traced stamps are those of the last launch
                pr, u, o, nr, dd = reps[i % a.rr]
                ctx.run(pr, epg.KERNEL_CFD_FLUX, u, o, nr, dd, 1)
            if a.chain:   # one more edge kernel: its stamps follow the finalise traced above
                pr, u, o, nr, dd = reps[(2 * a.rr) % a.rr]
                ctx.run_edges(pr, epg.KERNEL_CFD_FLUX, u, o, nr, dd)
            torch.cuda.synchronize()
        else:
            torch.cuda._sleep(2_000_000)               # keep the GPU busy while the host enqueues
            flush.fill_(rep & 255)
            ctx.run(plan, epg.KERNEL_CFD_FLUX, Un, out, nrm, dtn, 1)
            torch.cuda.synchronize()
        buf = np.zeros(1024 * niters * npts, dtype=np.uint64)
        epg.lib.epg_debug_trace(buf.ctypes.data, buf.size)
        buf = buf.astype(np.uint64)
        t = buf.reshape(1024, niters, npts)[:nblk, 0, :].astype(np.int64)
        epg.lib.epg_debug_trace_clear()
        base = t[:, 0][t[:, 0] > 0].min()
        if a.chain:
            f0 = buf.reshape(1024, niters, npts)[:, 14, 0].astype(np.int64)
            base = f0[f0 > 0].min()
        print(f"variant {v} rep {rep}: k_exec={plan.k_exec} CTAs traced={nblk}")
        for pt in range(npts):
            col = t[:, pt]
            col = col[col > 0]
            if col.size == 0:
                continue
            d = (col - base) / 1e3
            print(f"  pt{pt}: n={col.size:4d}  min {d.min():7.2f}  p10 {np.percentile(d, 10):7.2f}  "
                  f"p50 {np.percentile(d, 50):7.2f}  p90 {np.percentile(d, 90):7.2f}  max {d.max():7.2f} us")
        last_edge = t[:, 6][t[:, 6] > 0].max() if (t[:, 6] > 0).any() else base
        print(f"  last edge CTA done at {(last_edge - base) / 1e3:7.2f} us")
        fin = buf.reshape(1024, niters, npts)[:, 14, :3].astype(np.int64)
        fin = fin[fin[:, 0] > 0]
        if fin.size:
            for pt, name in enumerate(["finalise CTA start", "finalise wait released", "finalise CTA done"]):
                col = fin[:, pt][fin[:, pt] > 0]
                if col.size:
                    d = (col - base) / 1e3
                    print(f"  {name:24s} n={col.size:4d} min {d.min():7.2f} p50 {np.percentile(d, 50):7.2f} "
                          f"max {d.max():7.2f} us")
        for pa, pb in [(0, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 7), (0, 6), (0, 7)]:
            ok = (t[:, pa] > 0) & (t[:, pb] > 0)
            dd = (t[ok, pb] - t[ok, pa]) / 1e3
            if dd.size:
                print(f"  pt{pa}->pt{pb}: p10 {np.percentile(dd, 10):6.2f}  p50 {np.percentile(dd, 50):6.2f}  "
                      f"p90 {np.percentile(dd, 90):6.2f}  max {dd.max():6.2f} us")


if __name__ == "__main__":
    main()

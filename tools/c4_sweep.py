"""C4 (R-MAT scale 24 gather-scatter) parameter sweep on one GPU: partition size, execution
row cap and hub-split threshold; K back-to-back steps per setting (development tool).

    python tools/c4_sweep.py [--scale 24]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import synth as S  # noqa: E402
from paper_1605_02043_b200 import epg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--parts", default="1024,2048")
    ap.add_argument("--rows", default="1024,2048")
    ap.add_argument("--hubs", default="7,0,32")
    a = ap.parse_args()
    n, edges = S.rmat(a.scale)
    m = edges.shape[0]
    x = S.int_vector(1608, n, 0, 7)
    stream = torch.cuda.current_stream()
    ctx = epg.Context(0, stream)
    E = torch.from_numpy(edges).cuda()
    X = torch.from_numpy(x).cuda()
    for P in map(int, a.parts.split(",")):
        t0 = time.perf_counter()
        part, rank, rep = ctx.partition_rb(E, n, P, 1, 4096, ranked=True)
        tp = time.perf_counter() - t0
        k = epg.num_parts(m, P)
        for rows in map(int, a.rows.split(",")):
            for hub in a.hubs.split(","):
                os.environ["EPG_HUB_MIN"] = hub
                ctx.set_exec_limits(rows, 1280 if P > 1024 else 1024)
                L, plan = ctx.remap(E, n, part, k, halo_cap=rep.cut_cost, order_key=rank)
                xn = ctx.permute_rows(X, L.vertex_perm, epg.PERM_SCATTER)
                y = torch.empty_like(xn)
                for _ in range(3):
                    ctx.run(plan, epg.KERNEL_GATHER_SCATTER, xn, y, None, None, 1)
                torch.cuda.synchronize()
                ms = bench.timed_block(torch, stream, a.steps,
                                       lambda i: ctx.run(plan, epg.KERNEL_GATHER_SCATTER, xn, y, None, None, 1)) / a.steps
                print(json.dumps({"P": P, "exec_rows": rows, "hub_min": hub, "ms_per_step": ms, "k_exec": plan.k_exec,
                                  "hubs": plan.hubs, "R": rep.replication, "partition_s": tp}), flush=True)
                del L, plan, xn, y
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

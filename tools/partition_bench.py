"""EPG-RB partitioner timing and quality (P:907-910 weighs partition
time against kernel time). Prints one JSON line per run.

    python tools/partition_bench.py c3 [c4 c2 ...] [--leaf-parts 256] [--epg2]
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

import synth as S  # noqa: E402
from paper_1605_02043_b200 import epg  # noqa: E402


def graph(cfg):
    if cfg in ("c1", "c2", "c3"):
        M = S.config_mesh(cfg)
        return M.n, M.edges
    if cfg == "c4":
        return S.rmat(24)
    if cfg == "c5":
        n, e, _ = S.stencil2d_spmv(3536)
        return n, e
    raise SystemExit(cfg)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--leaf-parts", type=int, nargs="+", default=[256])
    ap.add_argument("--part-size", type=int, default=1024)
    ap.add_argument("--epg2", action="store_true", help="also time flat host EPG-2")
    ap.add_argument("--shards", type=int, default=1)
    a = ap.parse_args()
    ctx = epg.Context(0)
    for cfg in a.configs:
        t0 = time.perf_counter()
        n, e = graph(cfg)
        gen = time.perf_counter() - t0
        E = torch.from_numpy(e).cuda()
        for lp in a.leaf_parts:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            part, rep = ctx.partition_rb(E, n, a.part_size, a.shards, lp)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            print(json.dumps({"config": cfg, "method": "epg_rb", "leaf_parts": lp, "shards": a.shards,
                              "seconds": dt, "replication": rep.replication, "cut_cost": rep.cut_cost,
                              "load_count": rep.load_count, "touched": rep.touched, "m": len(e),
                              "host_cpus": os.cpu_count(), "gen_s": gen}), flush=True)
        if a.epg2:
            ctx.set_partition_method(2)
            t0 = time.perf_counter()
            part, rep = ctx.partition(E, n, a.part_size, a.shards)
            dt = time.perf_counter() - t0
            print(json.dumps({"config": cfg, "method": "epg2", "shards": a.shards, "seconds": dt,
                              "replication": rep.replication, "cut_cost": rep.cut_cost}), flush=True)


if __name__ == "__main__":
    main()

"""Summarise the ncu outputs of tools/profile_round.sh into profiles/ (committed evidence).

    python tools/summarize_ncu.py --config c2 --round r01

Writes profiles/<round>_<config>_launches.csv (kernel, launches, mean/median us, share),
profiles/<round>_<config>_variants.json (DRAM and L2->SM bytes per edge per schedule) and
profiles/<round>_<config>_full.txt (key metrics of the dominant kernel's full capture).
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import re
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def read_ncu_csv(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.reader(lines)
    hdr = None
    for r in rd:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            rows.append(dict(zip(hdr, r)))
    return rows


def short(name):
    m = re.match(r"(?:void )?(?:epg::)?([A-Za-z0-9_]+)(<[^(]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:60]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--round", default="r01")
    ap.add_argument("--m", type=int, default=None, help="edges of the config (for per-edge numbers)")
    a = ap.parse_args()
    g = os.path.join(ROOT, "gpurun_out")
    pre = os.path.join(ROOT, "profiles", f"{a.round}_{a.config}")
    m = a.m
    if m is None:
        sys.path.insert(0, ROOT)
        import synth
        m = synth.config_mesh(a.config).m
    # 1. launch list (optional: the bench's launch list is only taken for the headline config)
    lpath = os.path.join(g, f"launches_{a.config}.csv")
    rows = read_ncu_csv(lpath) if os.path.exists(lpath) else []
    per = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1000.0 if unit == "ns" else (v if unit == "us" else v * 1000.0)
        per.setdefault(short(r["Kernel Name"]), []).append(us)
    tot = sum(sum(v) for v in per.values())
    step = {k: v for k, v in per.items() if k.split("<")[0] in ("k_edge_occ", "k_finalise_rec", "k_finalise_rec16",
                                                                "k_finalise3")}
    step_tot = sum(statistics.median(v) for v in step.values()) or 1.0
    if not per:
        per = {}
    with open(pre + "_launches.csv", "w", newline="") if rows else open(os.devnull, "w") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "mean_us", "median_us", "total_us", "share_of_all", "share_of_step"])
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            ss = f"{statistics.median(v) / step_tot:.4f}" if k in step else ""
            w.writerow([k, len(v), f"{statistics.mean(v):.3f}", f"{statistics.median(v):.3f}", f"{sum(v):.3f}",
                        f"{sum(v) / tot:.4f}", ss])
    # 2. variants
    rows = read_ncu_csv(os.path.join(g, f"variants_{a.config}.csv"))
    kern = {}
    order = []
    step_kernels = ("k_edge_occ", "k_edge_tma", "k_edge_staged", "k_naive_edges", "k_naive_update",
                    "k_finalise_rec", "k_finalise_rec16", "k_finalise3", "k_finalise")
    for r in rows:
        base = short(r["Kernel Name"]).split("<")[0]
        if base not in step_kernels:
            continue
        key = (r["ID"], short(r["Kernel Name"]))
        if key not in kern:
            kern[key] = {}
            order.append(key)
        try:
            kern[key][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            pass
    log = open(os.path.join(g, f"variants_{a.config}.log")).read().split("\n")
    names = [ln.split(":")[0].replace("variant ", "") for ln in log if ln.startswith("variant ")]
    # launch order: ep (edge, finalise), default (edge, finalise), naive (edges, update)
    groups, cur = [], []
    for key in order:
        cur.append(key)
        if "finalise" in key[1] or "update" in key[1]:
            groups.append(cur)
            cur = []
    out = {"config": a.config, "m": m, "cache": "ncu default --cache-control all (cold L2 before each kernel)",
           "schedules": {}}
    for name, grp in zip(names, groups):
        d = {"kernels": [k[1] for k in grp]}
        dram = sum(kern[k].get("dram__bytes_read.sum", 0) + kern[k].get("dram__bytes_write.sum", 0) for k in grp)
        l2 = 32 * sum(kern[k].get("lts__t_sectors_srcunit_tex.sum", 0) for k in grp)
        t = sum(kern[k].get("gpu__time_duration.sum", 0) for k in grp)
        d.update({"dram_bytes": dram, "dram_bytes_per_edge": dram / m, "l2_sm_bytes": l2,
                  "l2_sm_bytes_per_edge": l2 / m, "time_us_cold": t / 1000.0})
        out["schedules"][name] = d
    ep_key = "ep" if "ep" in out["schedules"] else ("rb" if "rb" in out["schedules"] else None)
    if ep_key:
        ep = out["schedules"][ep_key]
        for other in ("default", "naive"):
            if other in out["schedules"]:
                o = out["schedules"][other]
                ep[f"dram_reduction_vs_{other}"] = o["dram_bytes"] / max(ep["dram_bytes"], 1)
                ep[f"l2_reduction_vs_{other}"] = o["l2_sm_bytes"] / max(ep["l2_sm_bytes"], 1)
    with open(pre + "_variants.json", "w") as f:
        json.dump(out, f, indent=1)
    # 3. full capture of the dominant kernel
    rep = os.path.join(g, f"full_edge_{a.config}.ncu-rep")
    if os.path.exists(rep):
        txt = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rr = list(csv.reader([ln for ln in raw.split("\n") if ln]))
        keys = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
                "launch__registers_per_thread", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                "lts__t_sectors_srcunit_tex.sum", "smsp__inst_executed.sum"]
        vals = {}
        if len(rr) >= 3:
            hdr, units, first = rr[0], rr[1], rr[2]
            for k in keys:
                if k in hdr:
                    vals[k] = first[hdr.index(k)] + " " + units[hdr.index(k)]
        with open(pre + "_full.txt", "w") as f:
            f.write(f"# ncu --set full of k_edge_occ ({a.config}, one cold launch)\n")
            for k, v in vals.items():
                f.write(f"{k} = {v}\n")
            f.write("\n")
            f.write(txt)
        traffic = None
        try:
            rb = float(vals["dram__bytes_read.sum"].split()[0].replace(",", ""))
            wb = float(vals["dram__bytes_write.sum"].split()[0].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rb *= scale.get(vals["dram__bytes_read.sum"].split()[1], 1)
            wb *= scale.get(vals["dram__bytes_write.sum"].split()[1], 1)
            traffic = rb + wb
        except (KeyError, IndexError, ValueError):
            pass
        with open(os.path.join(ROOT, "profiles", f"traffic_{a.config}.json"), "w") as f:
            json.dump({"config": a.config, "round": a.round, "kernel": "k_edge_occ<CfdFlux>",
                       "dram_bytes_per_launch": traffic,
                       "source": f"profiles/{a.round}_{a.config}_full.txt (ncu --set full, one cold launch)"}, f,
                      indent=1)
    if os.path.exists(pre + "_launches.csv"):
        print(open(pre + "_launches.csv").read())
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

"""Summarise an ncu source-page CSV (--page source --csv --print-source cuda|sass): top
lines by executed instructions, shared wavefronts (and excess) and stall samples."""
import csv, gzip, sys


def load(path):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as f:
        rows = list(csv.reader(f))
    out, fname, hdr = [], None, None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Name":
            fname = r[1].split("/")[-1]
            continue
        if r[0] in ("Line No", "Address"):
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        d["_file"] = fname
        out.append(d)
    return out, hdr


def num(d, k):
    try:
        return float(d.get(k, "0") or 0)
    except ValueError:
        return 0.0


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows, hdr = load(path)
    key = "Line No" if "Line No" in hdr else "Address"
    tot_i = sum(num(d, "Instructions Executed") for d in rows)
    tot_w = sum(num(d, "L1 Wavefronts Shared") for d in rows)
    tot_x = sum(num(d, "L1 Wavefronts Shared Excessive") for d in rows)
    tot_s = sum(num(d, "Warp Stall Sampling (All Samples)") for d in rows)
    print(f"total inst {tot_i:.4g}  shared wavefronts {tot_w:.4g} (excessive {tot_x:.4g})  stall samples {tot_s:.4g}")
    for metric in ("Instructions Executed", "L1 Wavefronts Shared Excessive", "Warp Stall Sampling (All Samples)"):
        print(f"\n== top by {metric}")
        for d in sorted(rows, key=lambda d: -num(d, metric))[:top]:
            print(f"{d['_file'][:18]:18s} {d[key]:>6s} inst {num(d,'Instructions Executed')/max(tot_i,1)*100:5.1f}% "
                  f"wf {num(d,'L1 Wavefronts Shared')/max(tot_w,1)*100:5.1f}% xs {num(d,'L1 Wavefronts Shared Excessive')/max(tot_x,1)*100:5.1f}% "
                  f"stall {num(d,'Warp Stall Sampling (All Samples)')/max(tot_s,1)*100:5.1f}% | {d['Source'].strip()[:90]}")


if __name__ == "__main__":
    main()

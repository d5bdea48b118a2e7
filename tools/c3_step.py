"""C3 step timing only (bench.py's C3 sub-record): python tools/c3_step.py [--comparators]"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1605_02043_b200 import epg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--comparators", action="store_true")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--order", choices=["growth", "id"], default="growth")
    ap.add_argument("--part-size", type=int, default=1024)
    ap.add_argument("--exec-rows", type=int, default=768)
    ap.add_argument("--leaf-parts", type=int, default=2048)
    a = ap.parse_args()
    args = argparse.Namespace(part_size=a.part_size, c3_steps=a.steps, no_comparators=not a.comparators, order=a.order,
                              exec_rows=a.exec_rows, c3_leaf_parts=a.leaf_parts)
    stream = torch.cuda.current_stream()
    ctx = epg.Context(0, stream)
    peak, _ = bench.measured_peaks()
    out = bench.run_c3(args, torch, epg, ctx, stream, peak)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Markdown table of tools/ab.sh results (mean over reps per workload and library).

    python tools/ab_report.py gpurun_out/ab_<tag>.jsonl [...]

Profiling aid only (not part of the product path).
"""
from __future__ import annotations

import json
import sys
from collections import defaultdict


def main():
    for path in sys.argv[1:]:
        acc = defaultdict(list)
        order = []
        for ln in open(path):
            d = json.loads(ln)
            b = d["line"]
            key = (b["config"]["workload"], d["lib"])
            if key not in acc:
                order.append(key)
            acc[key].append((b["value"], b["roofline"]["frac"]))
        print(f"### {path.split('/')[-1]}\n")
        print("| workload | library | reps | G DOF-stage/s | stage-kernel % of HBM |")
        print("|---|---|---|---|---|")
        for key in order:
            v = acc[key]
            print(f"| {key[0]} | {key[1]} | {len(v)} | {sum(x[0] for x in v) / len(v) / 1e9:.2f} | "
                  f"{100 * sum(x[1] for x in v) / len(v):.1f} |")
        print()


if __name__ == "__main__":
    main()

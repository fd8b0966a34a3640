#!/usr/bin/env python3
"""Markdown table of bench.py JSON lines (one per workload).

    python tools/bench_table.py gpurun_out/bench_all.jsonl [...]

Profiling aid only (not part of the product path).
"""
from __future__ import annotations

import json
import sys


def main():
    rows = []
    for path in sys.argv[1:]:
        for ln in open(path):
            ln = ln.strip()
            if not ln.startswith("{"):
                ln = ln[ln.find("{"):]
            if not ln:
                continue
            rows.append(json.loads(ln))
    print("| workload | DOF | G DOF-stage/s | ms/step | stage kernel ms | stage-kernel % of HBM peak | stage share of step |")
    print("|---|---|---|---|---|---|---|")
    for d in rows:
        r = d["roofline"]
        c = d["config"]
        print(f"| {c['workload']} | {c['dof']:,} | {d['value'] / 1e9:.1f} | {d['ms_per_step']:.2f} | "
              f"{r['stage_avg_ms']:.3f} | {100 * r['frac']:.1f} | {r['stage_share_of_step']:.3f} |")


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Markdown summary of tools/sweep.py outputs.

    python tools/sweep_report.py ORDER.json SHOCK.json > profiles/round1_sweeps.md

Profiling aid only (not part of the product path).
"""
from __future__ import annotations

import json
import sys


def order_table(d):
    out = ["## BASELINE configs[1]: isentropic vortex to t = 1, time to L2(rho) error (reading R8)", "",
           "Device seconds of `hom2d_step` (CUDA events) on the finest grid needed, log-log interpolated "
           "between bracketing grids; FV ladder NDoF-matched ((k+1)·n cells per side). CFL: Table 1 "
           "(P1/P2), the max-CFL protocol (P3/P4, `round1_cfl_protocol.md; P3/P4 ladders from 8² this round`). At these sizes every run is "
           "launch/latency-bound (<= ~10^6 DOF).", "",
           "| method | k | T(E=1e-4) s | T(E=2e-5) s | grids (n: L2, s) |", "|---|---|---|---|---|"]
    for r in d["results"]:
        t1, t2 = r.get("seconds_to_0.0001"), r.get("seconds_to_2e-05")
        f = lambda v: f"{v:.4f}" if v is not None else "n/a"  # noqa: E731
        grids = "; ".join(f"{g['n']}: {g['l2_rho']:.2e}, {1e3 * g['seconds']:.1f} ms" for g in r["grids"])
        out.append(f"| {r['method']} | {r['k']} | {f(t1)} | {f(t2)} | {grids} |")
    return out


def shock_table(d):
    out = ["## BASELINE configs[3]: radial shock tube to t = 0.25, limiter on (FV: MUSCL-2 for P1-matched, "
           "MUSCL-3 for P2-matched)", "",
           "Paper (K20c, P:1086-1116): at P2 / 1440k DoF CPR is 27 % faster per iteration than FV, DG 14 % "
           "slower; FV reaches t_end 25 % faster than CPR/SD.", "",
           "| k | DoF | method | cells/elements | CFL | steps | total s | ms/step |", "|---|---|---|---|---|---|---|---|"]
    for r in d["results"]:
        out.append(f"| {r['k']} | {r['dof']} | {r['method']} | {r['n']}^2 | {r['cfl']} | {r['steps']} | "
                   f"{r['seconds']:.3f} | {1e3 * r['seconds_per_step']:.3f} |")
    return out


def main():
    lines = ["# Round 1 sweeps (1 x B200) — `python tools/sweep.py order|shock`", ""]
    lines += order_table(json.load(open(sys.argv[1])))
    lines += [""]
    lines += shock_table(json.load(open(sys.argv[2])))
    print("\n".join(lines))


if __name__ == "__main__":
    main()

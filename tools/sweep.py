#!/usr/bin/env python3
"""BASELINE.json configs[1] and configs[3] on one GPU, through the public API.

  python tools/sweep.py order  [--out profiles/round1_sweep_order.json]
      isentropic vortex to t = 1, CPR/DG/NDG/SD P1..P4 and MUSCL-FV
      2/3 on a grid ladder until the L2 density error (R8) drops below 2e-5;
      per (method, k): error and device seconds per grid, and the time to reach
      E* = 1e-4 and 2e-5 by log-log interpolation between bracketing grids
      (the paper prints no error criterion).
  python tools/sweep.py shock  [--out profiles/round1_sweep_shock.json]
      radial shock tube to t = 0.25, transmissive, minmod limiter
      after every stage (HO) / MUSCL (FV), at the paper's DoF levels (Table 4:
      P1 160k / 640k, P2 360k / 1440k) with Table-4 CFLs: total device seconds,
      steps, seconds per step.

Times are CUDA-event device times of hom2d_step (t and dt stay on the device;
the host syncs once per 64 steps).  CFL values: Table 1 and Table 4
(P:1048-1066); P3/P4 provisional.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CFL_SMOOTH = {("cpr", 1): 0.24, ("ndg", 1): 0.24, ("dg", 1): 0.24, ("sd", 1): 0.3,
              ("cpr", 2): 0.13, ("ndg", 2): 0.13, ("dg", 2): 0.13, ("sd", 2): 0.2,
              # P3/P4: not in Table 1; SURVEY Q23's 1/(2k+1) fit (0.10 / 0.08) is unstable for
              # CPR P3 on the vortex, so start lower; an unstable run halves the CFL (max-CFL
              # protocol direction) and is reported
              ("cpr", 3): 0.08, ("ndg", 3): 0.08, ("dg", 3): 0.08, ("sd", 3): 0.10,
              ("cpr", 4): 0.05, ("ndg", 4): 0.05, ("dg", 4): 0.05, ("sd", 4): 0.06,
              ("fv", 1): 0.37, ("fv", 2): 0.37}
LADDER = [20, 28, 40, 57, 80, 113, 160, 226, 320, 453, 640, 905, 1280, 1810, 2560]
TARGETS = (1e-4, 2e-5)


def run_case(P, torch, method, k, n, cfl, case, t_end, box, bc, limiter):
    cfg = P.make_config(n, n, method=method, k=k, cfl=cfl, box=box, bc=bc, limiter=limiter)
    s = P.Solver(cfg)
    s.init_case(case)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    t, steps = s.step(10 ** 7, t_end)
    e1.record(stream)
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) / 1e3
    err = s.error(P.VORTEX, 0)[1] if case == P.VORTEX else None
    npe = 1 if method == "fv" else (k + 1) ** 2
    s.close()
    return {"method": method, "k": k, "n": n, "dof": n * n * npe, "cfl": cfl, "t": t, "steps": steps,
            "seconds": sec, "l2_rho": err, "dof_stage_per_s": n * n * npe * 3 * steps / sec if sec > 0 else None}


def time_to_error(rows, target):
    for a, b in zip(rows, rows[1:]):
        if a["l2_rho"] >= target >= b["l2_rho"]:
            la, lb = math.log(a["l2_rho"]), math.log(b["l2_rho"])
            w = (math.log(target) - la) / (lb - la) if lb != la else 0.0
            return math.exp(math.log(a["seconds"]) + w * (math.log(b["seconds"]) - math.log(a["seconds"])))
    if rows and rows[0]["l2_rho"] <= target:
        return rows[0]["seconds"]
    return None


def order_sweep(P, torch, out):
    res = []
    combos = [(m, k) for m in ("cpr", "dg", "ndg", "sd") for k in (1, 2, 3, 4)] + [("fv", 1), ("fv", 2)]
    for method, k in combos:
        rows = []
        cfl = CFL_SMOOTH[(method, k)]
        for n in LADDER:
            nn = n * (k + 1) if method == "fv" else n  # FV: NDoF-matched ladder
            while True:
                try:
                    r = run_case(P, torch, method, k, nn, cfl, P.VORTEX, 1.0, (-5.0, 5.0, -5.0, 5.0), 0, 0)
                    break
                except P.NonPhysicalState:
                    print(json.dumps({"method": method, "k": k, "n": nn, "cfl": cfl, "unstable": True}), flush=True)
                    cfl *= 0.5
            rows.append(r)
            print(json.dumps(r), flush=True)
            if r["l2_rho"] <= min(TARGETS) * 0.7 or r["seconds"] > 30:
                break
        summary = {"method": method, "k": k, "grids": rows}
        for tgt in TARGETS:
            summary[f"seconds_to_{tgt:g}"] = time_to_error(rows, tgt)
        res.append(summary)
        print(json.dumps({kk: v for kk, v in summary.items() if kk != "grids"}), flush=True)
    with open(out, "w") as f:
        json.dump({"case": "isentropic vortex t=1", "targets": TARGETS, "results": res}, f, indent=1)


def shock_sweep(P, torch, out):
    # Table 4: DoF levels and CFLs; FV matched by NDoF, MUSCL-2 (P1) / MUSCL-3 (P2)
    cfl = {("cpr", 1): 0.2, ("ndg", 1): 0.2, ("sd", 1): 0.27, ("dg", 1): 0.2, ("fv", 1): 0.58,
           ("cpr", 2): 0.1, ("ndg", 2): 0.1, ("sd", 2): 0.18, ("dg", 2): 0.08, ("fv", 2): 0.54}
    res = []
    for k, sizes in ((1, (200, 400)), (2, (200, 400))):
        for n in sizes:
            for method in ("cpr", "ndg", "sd", "dg", "fv"):
                nn = n * (k + 1) if method == "fv" else n
                r = run_case(P, torch, method, k, nn, cfl[(method, k)], P.SHOCK, 0.25, (-1.0, 1.0, -1.0, 1.0), 1,
                             0 if method == "fv" else 1)
                r["seconds_per_step"] = r["seconds"] / max(r["steps"], 1)
                res.append(r)
                print(json.dumps(r), flush=True)
    with open(out, "w") as f:
        json.dump({"case": "radial shock tube t=0.25, limiter on", "results": res}, f, indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["order", "shock"])
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    import paper_1709_01619_b200 as P
    from paper_1709_01619_b200 import build
    build.build()
    torch.cuda.set_device(0)
    out = args.out or os.path.join(ROOT, "profiles", f"round1_sweep_{args.what}.json")
    if args.what == "order":
        order_sweep(P, torch, out)
    else:
        shock_sweep(P, torch, out)


if __name__ == "__main__":
    main()

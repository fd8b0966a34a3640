#!/usr/bin/env python3
"""Table 1 under the literal max-CFL protocol of P:875-878 ("A new
simulation is completed at a value of 0.5*CFL of the previous ... If the percent
error between these two errors is less than 0.1 %, the CFL is termed the maximum
CFL"), read as a halving search: a printed value c is what that search returns
when started at 2c iff the run at c passes (L2(rho) error at t = 1 within 0.1 %
of the run at c/2) and the run at 2c does not (non-physical, or the change is
>= 0.1 %).  Runs the CPU oracle at every DoF level of Table 1 (~4 min on one
core) and writes a markdown table.

    python tools/cfl_halving.py [--out profiles/round2_cfl_halving.md]

Test infrastructure (calls oracle/), not part of the product path.
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import oracle  # noqa: E402
from sweep import TABLE1  # noqa: E402


def change(method, k, n, c):
    """|e(c) - e(c/2)| / e(c/2) of the vortex L2(rho) error at t = 1, or None if
    the run at c is non-physical"""
    def err(cfl):
        cf = oracle.config(nx=n, ny=n, method=method, k=k, cfl=cfl)
        try:
            q, t, _ = oracle.run(cf, oracle.init_case(cf), 10 ** 7, 1.0)
        except FloatingPointError:
            return None
        e = oracle.error(cf, q, t)[1]
        return e if math.isfinite(e) else None
    e1 = err(c)
    if e1 is None:
        return None
    return abs(e1 - err(c / 2)) / err(c / 2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "round2_cfl_halving.md"))
    args = ap.parse_args()
    lines = ["# Table 1 under the halving reading of the max-CFL protocol (`tools/cfl_halving.py`, CPU oracle)", "",
             "Cell: printed CFL c, change at c, change at 2c (in %; `blow-up` = non-physical).",
             "`ok` = the halving search started at 2c returns c (c passes, 2c fails).", "",
             "| k | DoF | CPR | NDG | SD | DG | FV |", "|---|---|---|---|---|---|---|"]
    n_ok = n_all = 0
    for k in (1, 2):
        for i, dof in enumerate(TABLE1[k]["dof"]):
            cells = []
            for m in ("cpr", "ndg", "sd", "dg", "fv"):
                n = int(round(math.sqrt(dof if m == "fv" else dof / (k + 1) ** 2)))
                c = TABLE1[k][m][i]
                a, b = change(m, k, n, c), change(m, k, n, 2 * c)
                ok = a is not None and a < 1e-3 and (b is None or b >= 1e-3)
                n_ok += ok
                n_all += 1
                fb = "blow-up" if b is None else f"{100 * b:.3f}"
                cells.append(f"{c}: {100 * a:.4f} / {fb} {'ok' if ok else '**no**'}")
            lines.append(f"| {k} | {dof} | " + " | ".join(cells) + " |")
            print(lines[-1], flush=True)
    lines += ["", f"{n_ok} of {n_all} printed values are the halving search's answer from twice their value."]
    with open(args.out, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()

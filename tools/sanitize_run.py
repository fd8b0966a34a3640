#!/usr/bin/env python3
"""A small run of every stage-kernel family for compute-sanitizer:

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck \\
        python tools/sanitize_run.py [--quick]

Every method x order on a ragged grid (several strips / marches, both BCs):
init, 3 SSP-RK3 steps (stage kernels incl. the dt / non-physical epilogue, k_dt),
one residual, the error reductions; the limiter kernels on the shock tube; the
FV odd-width (CTA) and even-width (warp) kernels; DG over-integration; the
multi-GPU stage path through the self-exchange and 1-rank NCCL test modes.
Profiling aid only (no oracle, no assertions beyond the library's own statuses).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1709_01619_b200 as P
    quick = "--quick" in sys.argv
    torch.cuda.set_device(0)
    cases = [(m, k) for m in ("cpr", "ndg", "dg", "sd") for k in (1, 2, 3, 4)] + [("fv", 1), ("fv", 2)]
    if quick:
        cases = [("cpr", 3), ("dg", 2), ("sd", 4), ("ndg", 1), ("fv", 1), ("fv", 2)]
    n_run = 0
    for method, k in cases:
        for bc in (0, 1):
            for nx, ny in ((19, 13), (66, 9)) if method != "fv" else ((45, 21), (130, 9)):
                # the vortex on both boundary conditions (the unlimited shock tube is
                # not physical for long); the shock tube runs with the limiter below
                s = P.Solver(P.make_config(nx, ny, method=method, k=k, bc=bc, cfl=0.05))
                s.init_case(P.VORTEX)
                s.step(3)
                q = s.get_state(torch.empty(s.n_values, dtype=torch.float64, device="cuda"))
                s.residual(q)
                s.error(P.VORTEX, 0)
                s.close()
                n_run += 1
        if method != "fv" and k <= 2:  # limiter kernels (averages fused / k_avg, k_limit, k_lambda)
            s = P.Solver(P.make_config(24, 18, method=method, k=k, bc=1, box=(-1.0, 1.0, -1.0, 1.0), cfl=0.05,
                                       limiter=1, record_decisions=1))
            s.init_case(P.SHOCK)
            s.step(3)
            s.decisions()
            s.close()
            n_run += 1
    for k in (1, 3):  # DG over-integration
        s = P.Solver(P.make_config(17, 11, method="dg", k=k, cfl=0.05, dg_overintegrate=1))
        s.init_case(P.VORTEX)
        s.step(2)
        s.close()
    s = P.Solver(P.make_config(40, 30, method="fv", k=2, cfl=0.3, fv_error_recon=1))
    s.init_case(P.VORTEX)
    s.error(P.VORTEX, 1)
    s.close()
    for sx in ("1", "2", "3"):  # the multi-GPU stage path on one GPU (3: peer-memory halo)
        os.environ["HOM2D_SELF_EXCHANGE"] = sx
        for method, k in (("cpr", 3), ("fv", 1), ("dg", 2)):
            s = P.Solver(P.make_config(23, 14, method=method, k=k, cfl=0.05, limiter=1 if method == "dg" else 0))
            s.init_case(P.VORTEX)
            s.step(3)
            s.close()
        os.environ.pop("HOM2D_SELF_EXCHANGE")
    torch.cuda.synchronize()
    print(f"sanitize_run ok ({n_run} configurations)")


if __name__ == "__main__":
    main()

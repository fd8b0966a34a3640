#!/usr/bin/env python3
"""Paper-size (latency-bound) grids: device microseconds per SSP-RK3 step of
hom2d_step against the launch floor.

    python tools/small_grids.py [--out gpurun_out/small_grids.json]

For each (method, k): the per-step time on a 2x2-element grid (the kernels do
next to no work: the floor of the step's launch chain -- 3 stage kernels with
programmatic dependent launch, the dt fused into stages 1-2; HOM2D_NO_DTFUSE=1
for the k_dt chain), on the paper's grids (20^2, P3/P4 also
8^2; FV NDoF-matched) and on 80^2, each in three launch modes: eager launches,
CUDA graphs after 2048 eager steps (the default), graphs from the first step
(HOM2D_GRAPH_AFTER=0, HOM2D_GRAPH_MIN_BATCH=1).  Runs of 512 steps after a
64-step warm-up; CUDA events on the library's stream.  Profiling aid only.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

MODES = {"eager": {"HOM2D_NO_GRAPH": "1"},
         "default": {},
         "graph_first": {"HOM2D_GRAPH_AFTER": "0", "HOM2D_GRAPH_MIN_BATCH": "1"}}


def per_step_us(P, torch, method, k, n, steps=512, cold=False):
    s = P.Solver(P.make_config(n, n, method=method, k=k, cfl=0.05 if method != "fv" else 0.3))
    s.init_case(P.VORTEX)
    stream = torch.cuda.current_stream()
    if not cold:
        s.step(64)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    _, done = s.step(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    s.close()
    return 1e3 * e0.elapsed_time(e1) / done


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "small_grids.json"))
    args = ap.parse_args()
    import torch
    import paper_1709_01619_b200 as P
    torch.cuda.set_device(0)
    combos = [("cpr", 1), ("cpr", 3), ("cpr", 4), ("dg", 2), ("sd", 3), ("ndg", 2), ("fv", 1), ("fv", 2)]
    rows = []
    for mode, env in MODES.items():
        for key in ("HOM2D_NO_GRAPH", "HOM2D_GRAPH_AFTER", "HOM2D_GRAPH_MIN_BATCH"):
            os.environ.pop(key, None)
        os.environ.update(env)
        for method, k in combos:
            grids = [2, 20, 80] if method != "fv" else [4, 20 * (k + 1), 80 * (k + 1)]
            if method != "fv" and k >= 3:
                grids.insert(1, 8)
            for n in grids:
                per_step_us(P, torch, method, k, n, steps=16)  # lazy module load
                us = per_step_us(P, torch, method, k, n)
                cold = per_step_us(P, torch, method, k, n, steps=128, cold=True)
                rows.append({"mode": mode, "method": method, "k": k, "n": n, "us_per_step": us,
                             "us_per_step_first_128_cold": cold})
                print(json.dumps(rows[-1]), flush=True)
    with open(args.out, "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()

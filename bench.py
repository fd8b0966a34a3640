#!/usr/bin/env python3
"""Benchmark of the hot path: SSP-RK3 steps of the 2-D Euler CPR P3 isentropic
vortex on 4096x4096 elements (BASELINE.json north_star; 268,435,456 DOF, fp64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--workload cpr_p3_4096|cpr_p3_2048|cpr_p2_8192w|fv2_8192w]
    torchrun --nproc-per-node N bench.py --gpus N ...   (N > 1: y-strips over NCCL)

Metric: DOF-stage updates per second: N_DOF(points) x 3 RK stages
x K steps / seconds, whole job.  One "step" = one SSP-RK3 step = the whole hot
path (3 fused residual+RK stage kernels, the dt bookkeeping, the wave-speed
max-reduction and, at N > 1, the halo exchange and the dt allreduce).
Inputs (8.6 GB/state array at the default workload) are far larger than the
126 MB L2, so no flush is needed between steps.

Prints ONE JSON line on rank 0.  `--impl reference` times the CPU oracle (the
reference arm of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (method, k, nx, ny, cfl, weak)
    "cpr_p3_4096": ("cpr", 3, 4096, 4096, 0.08, False),   # north star
    "cpr_p3_2048": ("cpr", 3, 2048, 2048, 0.08, False),   # BASELINE configs[2] (d3)
    "cpr_p2_8192w": ("cpr", 2, 8192, 1024, 0.13, True),   # configs[4], per-GPU strip (d5)
    "fv2_8192w": ("fv", 1, 8192, 1024, 0.37, True),       # configs[4], per-GPU strip (d5)
    # per-method throughput at matched DOF (268M points; FV 16384^2 cells)
    "ndg_p3_4096": ("ndg", 3, 4096, 4096, 0.08, False),
    "dg_p3_4096": ("dg", 3, 4096, 4096, 0.08, False),
    "sd_p3_4096": ("sd", 3, 4096, 4096, 0.10, False),
    "cpr_p2_4096": ("cpr", 2, 4096, 4096, 0.13, False),
    "cpr_p1_8192": ("cpr", 1, 8192, 8192, 0.24, False),
    "cpr_p4_4096": ("cpr", 4, 4096, 4096, 0.05, False),
    "ndg_p1_8192": ("ndg", 1, 8192, 8192, 0.24, False),
    "ndg_p2_4096": ("ndg", 2, 4096, 4096, 0.13, False),
    "ndg_p4_4096": ("ndg", 4, 4096, 4096, 0.05, False),
    "dg_p1_8192": ("dg", 1, 8192, 8192, 0.24, False),
    "dg_p2_4096": ("dg", 2, 4096, 4096, 0.13, False),
    "dg_p4_4096": ("dg", 4, 4096, 4096, 0.05, False),
    "sd_p1_8192": ("sd", 1, 8192, 8192, 0.3, False),
    "sd_p2_4096": ("sd", 2, 4096, 4096, 0.2, False),
    "sd_p4_4096": ("sd", 4, 4096, 4096, 0.08, False),
    "fv2_16384": ("fv", 1, 16384, 16384, 0.37, False),
    "fv3_16384": ("fv", 2, 16384, 16384, 0.37, False),
    # limiter-on throughput: the radial shock tube scaled up,
    # transmissive, minmod detection + limiting after every stage, Table 4 CFLs
    "cpr_p1_shock_4096": ("cpr", 1, 4096, 4096, 0.2, False, "shock"),
    "cpr_p2_shock_4096": ("cpr", 2, 4096, 4096, 0.1, False, "shock"),
    "dg_p1_shock_4096": ("dg", 1, 4096, 4096, 0.2, False, "shock"),
    "sd_p1_shock_4096": ("sd", 1, 4096, 4096, 0.27, False, "shock"),
    "fv2_shock_8192": ("fv", 1, 8192, 8192, 0.58, False, "shock"),
}


def workload(wl):
    """(method, k, nx, ny, cfl, weak, case) of a bench workload."""
    w = WORKLOADS[wl]
    return (*w[:6], w[6] if len(w) > 6 else "vortex")
BYTES_PER_DOF_STEP = 256.0   # algorithmic HBM bytes: stage 1 64 B, stages 2/3 96 B


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_info():
    """lscpu model and core counts of the host, and the CPUs this process may use."""
    info = {"model": "unknown"}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        keys = {"Model name:": "model", "Socket(s):": "sockets", "Core(s) per socket:": "cores_per_socket",
                "Thread(s) per core:": "threads_per_core", "CPU(s):": "cpus"}
        for line in out.splitlines():
            for k, name in keys.items():
                if line.startswith(k):
                    v = line.split(":", 1)[1].strip()
                    info[name] = int(v) if v.isdigit() else v
    except Exception:
        pass
    info["usable_cpus"] = usable_cpus()
    return info


def usable_cpus():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


DATA = {"vortex": "synthetic (closed-form isentropic vortex, P:897-913)",
        "shock": "synthetic (radial shock tube, P:1043-1047, scaled up; limiter on)"}


def oracle_rate(method, k, nx, ny, cfl, steps, case="vortex", threads=1):
    """The CPU oracle as it stands, DOF-stage/s on a sample grid, on `threads`
    host threads (OpenMP over elements; bitwise the single-thread result)."""
    import oracle
    oracle.set_threads(threads)
    if case == "shock":
        cfg = oracle.config(nx=nx, ny=ny, method=method, k=k, cfl=cfl, bc=oracle.TRANSMISSIVE,
                            box=(-1.0, 1.0, -1.0, 1.0), limiter=1)
        q = oracle.init_case(cfg, oracle.SHOCK)
    else:
        cfg = oracle.config(nx=nx, ny=ny, method=method, k=k, cfl=cfl)
        q = oracle.init_case(cfg)
    t0 = time.perf_counter()
    oracle.run(cfg, q, steps)
    dt = time.perf_counter() - t0
    oracle.set_threads(1)
    ndof = nx * ny * (1 if method == "fv" else (k + 1) ** 2)
    return ndof * 3 * steps / dt, dt


def reference_arm(args, wl):
    """--impl reference: the oracle timed on the host, bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    method, k, nx, ny, cfl, weak, case = workload(wl)
    nth = usable_cpus()
    oracle.set_threads(nth)
    sn = 256 if method != "fv" else 1024
    if case == "shock":
        cfg = oracle.config(nx=sn, ny=sn, method=method, k=k, cfl=cfl, bc=oracle.TRANSMISSIVE,
                            box=(-1.0, 1.0, -1.0, 1.0), limiter=1)
        q = oracle.init_case(cfg, oracle.SHOCK)
    else:
        cfg = oracle.config(nx=sn, ny=sn, method=method, k=k, cfl=cfl)
        q = oracle.init_case(cfg)
    for _ in range(args.warmup):
        q, _, _ = oracle.run(cfg, q, 1)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        q, _, _ = oracle.run(cfg, q, 1)
    el = time.perf_counter() - t0
    oracle.set_threads(1)
    ndof = sn * sn * (1 if method == "fv" else (k + 1) ** 2)
    v = ndof * 3 * args.steps / el
    sample = (f"{method.upper()} P{k} {case} {sn}x{sn} (sample of {nx}x{ny}), 1 SSP-RK3 step per bench step, "
              f"{nth} OpenMP threads")
    line = {"impl": "reference", "metric": "fp64 DOF-stage updates/s", "value": v, "unit": "DOF-stage/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f64",
            "data": DATA[case],
            "config": {"workload": f"{wl} (oracle sample {sn}x{sn})", "method": method, "k": k, "nx": sn, "ny": sn},
            "cpu_baseline": {"value": v, "unit": "DOF-stage/s", "cores": nth, "kind": "oracle", "sample": sample,
                             "cpu": cpu_info()},
            "e2e": {"value": v, "unit": "DOF-stage/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# CFL of the smooth problem: Table 1 for P1/P2, the max-CFL protocol for P3/P4
# (profiles/round1_cfl_protocol.md); FV Table 1's smallest value
TTE_CFL = {("cpr", 1): 0.24, ("ndg", 1): 0.24, ("dg", 1): 0.24, ("sd", 1): 0.3,
           ("cpr", 2): 0.13, ("ndg", 2): 0.13, ("dg", 2): 0.13, ("sd", 2): 0.2,
           ("cpr", 3): 0.09, ("ndg", 3): 0.09, ("dg", 3): 0.09, ("sd", 3): 0.09,
           ("cpr", 4): 0.05, ("ndg", 4): 0.06, ("dg", 4): 0.04, ("sd", 4): 0.03,
           ("fv", 1): 0.37, ("fv", 2): 0.37}
TTE_TARGETS = (1e-4, 2e-5)


def time_to_error(P, torch, method, k, stream, max_seconds=20.0):
    """The second half of the BASELINE metric (configs[1]): isentropic vortex to
    t = 1 on a grid ladder (FV NDoF-matched), L2(rho) error (reading
    R8) and device seconds of hom2d_step per grid; T(E*) by log-log interpolation
    between the bracketing grids (E* = 1e-4, 2e-5).  One GPU."""
    ladder = [20, 28, 40, 57, 80, 113, 160, 226, 320, 453, 640, 905, 1280, 1810, 2560]
    if method != "fv" and k >= 3:  # P3/P4 reach 1e-4 below 20^2: start at 8^2 so T(E*) is interpolated
        ladder = [8, 10, 12, 14, 17, 20, 24, 28, 34, 40, 48, 57, 68, 80, 96, 113]
    rows, spent = [], 0.0
    for n in ladder:
        nn = n * (k + 1) if method == "fv" else n
        s = P.Solver(P.make_config(nn, nn, method=method, k=k, cfl=TTE_CFL[(method, k)]), stream=stream)
        s.init_case(P.VORTEX)
        if not rows:  # load the kernels once, untimed (lazy module loading)
            s.step(1)
            s.init_case(P.VORTEX)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        t, steps = s.step(10 ** 7, 1.0)
        e1.record(stream)
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) / 1e3
        err = s.error(P.VORTEX, 0)[1]
        s.close()
        rows.append({"n": nn, "l2_rho": err, "seconds": sec, "steps": steps})
        spent += sec
        if err <= min(TTE_TARGETS) or spent > max_seconds:
            break
    out = {"case": "isentropic vortex to t = 1 (BASELINE configs[1])", "cfl": TTE_CFL[(method, k)], "grids": rows}
    for tgt in TTE_TARGETS:
        val = None
        for a_, b_ in zip(rows, rows[1:]):
            if a_["l2_rho"] >= tgt >= b_["l2_rho"]:
                la, lb = math.log(a_["l2_rho"]), math.log(b_["l2_rho"])
                w = (math.log(tgt) - la) / (lb - la) if lb != la else 0.0
                val = math.exp(math.log(a_["seconds"]) + w * (math.log(b_["seconds"]) - math.log(a_["seconds"])))
                break
        if val is None and rows and rows[0]["l2_rho"] <= tgt:
            val = rows[0]["seconds"]
        out[f"seconds_to_{tgt:g}"] = val
    return out


def traffic_from_profiles(wl):
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)
        return d.get(wl)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="hom2d", choices=["hom2d", "reference"])
    ap.add_argument("--workload", default="cpr_p3_4096", choices=sorted(WORKLOADS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tte", action="store_true", help="skip the time-to-error ladder")
    ap.add_argument("--no-weak", action="store_true", help="skip the weak-scaling workloads (configs[4])")
    ap.add_argument("--halo", default="nccl", choices=["nccl", "peer"],
                    help="N > 1: strip halo by NCCL send/recv (default) or by the peer-memory pull (hom2d_peer_connect)")
    args = ap.parse_args()
    assert args.warmup >= 3, "timing rules: W >= 3"
    wl = args.workload
    if args.impl == "reference":
        return reference_arm(args, wl)

    import torch
    import torch.distributed as dist

    import paper_1709_01619_b200 as P
    from paper_1709_01619_b200 import build

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE {world}"
    if rank == 0:
        build.build()
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL's communicator-init lines (nranks, ring/tree/NVLS setup) on stderr, for
        # the driver's check of the communicator size; INIT only, to keep them short
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        dist.barrier()
    method, k, nx, ny, cfl, weak, case = workload(wl)
    if weak:
        ny = ny * world
    nid = None
    if world > 1:
        obj = [P.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    stream = torch.cuda.current_stream()
    if case == "shock":
        cfg = P.make_config(nx, ny, method=method, k=k, cfl=cfl, bc=P.TRANSMISSIVE, box=(-1.0, 1.0, -1.0, 1.0),
                            limiter=0 if method == "fv" else 1)
    else:
        cfg = P.make_config(nx, ny, method=method, k=k, cfl=cfl)
    s = P.Solver(cfg, rank=rank, nranks=world, device=local, stream=stream, nccl_id=nid)
    if world > 1 and args.halo == "peer":
        P.connect_peers(s)
    s.init_case(P.SHOCK if case == "shock" else P.VORTEX)
    npe = 1 if method == "fv" else (k + 1) ** 2
    ndof_global = nx * ny * npe
    ndof_local = nx * s.nrows * npe

    def barrier_sync():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warm-up --------------------------------------------------------------
    s.step(args.warmup)
    barrier_sync()

    # ---- timed region (device): K steps, CUDA events on the library's stream --
    s.stage_timing(3 * args.steps + 8)
    launches0 = s.launch_count()
    clk = ClockSampler(local)
    clk.start()
    barrier_sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    s.step(args.steps)
    e1.record(stream)
    barrier_sync()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    stage_ms, n_stage = s.stage_time()
    gpu_launches = s.launch_count() - launches0
    t_ms = torch.tensor([ms, stage_ms / max(n_stage, 1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    ms, stage_avg_ms = float(t_ms[0]), float(t_ms[1])
    value = ndof_global * 3 * args.steps / (ms * 1e-3)

    # ---- e2e through the public API with host buffers ----------------------------
    e2e = None
    if not args.no_e2e:
        host_in = torch.empty(4 * ndof_local, dtype=torch.float64, pin_memory=True)
        host_out = torch.empty(4 * ndof_local, dtype=torch.float64, pin_memory=True)
        s.get_state(host_in)
        barrier_sync()
        t0 = time.perf_counter()
        s.set_state(host_in)          # H2D copy of the initial state (pinned host memory)
        for _ in range(args.steps):   # one public call per step: H2D of t_end, D2H of {t, dt, steps, flags}
            s.step(1)
        s.get_state(host_out)         # D2H read of the final state
        barrier_sync()
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        nbytes = 4 * ndof_local * 8
        e2e = {"value": ndof_global * 3 * args.steps / float(el[0]), "unit": "DOF-stage/s",
               "h2d_bytes_per_step": nbytes / args.steps + 8, "d2h_bytes_per_step": nbytes / args.steps + 40,
               "note": "hom2d_set_state(pinned host) + K x hom2d_step(1) (each: t_end H2D 8 B, clock + "
                       "non-physical flag D2H 40 B, host sync) + hom2d_get_state(pinned host); state bytes "
                       "amortised over the K steps"}

    # ---- roofline of the dominant kernel (the fused RK-stage kernel) --------------
    peak, peak_src = peaks()
    achieved = ndof_local * (BYTES_PER_DOF_STEP / 3.0) / (stage_avg_ms * 1e-3) / 1e9
    tr = traffic_from_profiles(wl)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": tr, "peak_source": peak_src, "kernel": (f"gll_stage_kernel<{method},{k}>" if method in ("cpr", "ndg") else
                           f"fv_warp_kernel<{k}>" if method == "fv" else f"gl_stage_kernel<{method},{k}>"),
                "stage_avg_ms": stage_avg_ms, "bytes_per_launch": ndof_local * BYTES_PER_DOF_STEP / 3.0,
                "stage_share_of_step": 3 * stage_avg_ms / (ms / args.steps)}

    tte = None
    if world == 1 and case == "vortex" and not args.no_tte:
        tte = time_to_error(P, torch, method, k, stream)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the oracle on all usable host threads (the reported value) and
        # on one thread (definitional), same sample; ~10-20 s of CPU work in total
        nth = usable_cpus()
        sn = 768 if method != "fv" else 3072
        v, el = oracle_rate(method, k, sn, sn, cfl, 6, case, threads=nth)
        sn1 = 384 if method != "fv" else 1536
        v1, el1 = oracle_rate(method, k, sn1, sn1, cfl, 4, case, threads=1)
        cpu = {"value": v, "unit": "DOF-stage/s", "cores": nth, "kind": "oracle",
               "sample": f"{method.upper()} P{k} {case} {sn}x{sn} elements, 6 SSP-RK3 steps on {nth} OpenMP "
                         f"threads ({el:.1f} s)",
               "single_thread": {"value": v1, "sample": f"{sn1}x{sn1} elements, 4 steps ({el1:.1f} s)"},
               "cpu": cpu_info()}

    # ---- the weak-scaling workloads (BASELINE configs[4]: per GPU 8192 x 1024
    # elements of CPR P2 / MUSCL-2 cells, y-strips) measured in the same run, so a
    # scaling sweep over N yields both curves; device time, max over ranks -------
    weak_lines = None
    if not args.no_weak and not weak:
        weak_lines = []
        for wwl in ("cpr_p2_8192w", "fv2_8192w"):
            wm, wk, wnx, wny, wcfl, _, _ = workload(wwl)
            wny *= world
            wid = None
            if world > 1:  # a fresh NCCL unique id per communicator (an id initialises one communicator only)
                obj = [P.nccl_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(obj, src=0)
                wid = obj[0]
            ws = P.Solver(P.make_config(wnx, wny, method=wm, k=wk, cfl=wcfl), rank=rank, nranks=world, device=local,
                          stream=stream, nccl_id=wid)
            if world > 1 and args.halo == "peer":
                P.connect_peers(ws)
            ws.init_case(P.VORTEX)
            ws.step(args.warmup)
            barrier_sync()
            w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            w0.record(stream)
            ws.step(args.steps)
            w1.record(stream)
            barrier_sync()
            wt = torch.tensor([w0.elapsed_time(w1)], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(wt, op=dist.ReduceOp.MAX)
            wnpe = 1 if wm == "fv" else (wk + 1) ** 2
            weak_lines.append({"workload": wwl, "scaling": "weak", "nx": wnx, "ny": wny,
                               "dof": wnx * wny * wnpe, "value": wnx * wny * wnpe * 3 * args.steps / (float(wt[0]) * 1e-3),
                               "unit": "DOF-stage/s", "ms_per_step": float(wt[0]) / args.steps})
            ws.close()

    if rank == 0:
        line = {"metric": "fp64 DOF-stage updates/s", "value": value, "unit": "DOF-stage/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "weak" if weak else "strong", "vs_baseline": None,
                "dtype": "f64", "data": DATA[case],
                "config": {"workload": wl, "method": method, "k": k, "nx": nx, "ny": ny, "dof": ndof_global,
                           "case": ("isentropic vortex, periodic" if case == "vortex" else
                                    "radial shock tube, transmissive, minmod limiter every stage"),
                           "cfl": cfl, "parallelism": f"ystrip{world}",
                           "halo": (args.halo if world > 1 else "none (1 GPU: periodic wrap in place)"),
                           "l2_flush": f"none needed: {4 * ndof_global * 8 / 1e9:.2f} GB/state array >> 126 MB L2"},
                "e2e": e2e, "gpu_launches": gpu_launches, "roofline": roofline, "cpu_baseline": cpu,
                "time_to_error": tte,
                "weak_scaling_workloads": weak_lines,
                "clocks": clocks,
                "hbm_frac_end_to_end": value * BYTES_PER_DOF_STEP / 3.0 / 1e9 / world / peak}
        print(json.dumps(line), flush=True)
    s.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""bench.py's contract on the host (no GPU): the reference arm (the CPU oracle
timed on a bounded sample of the workload) prints one JSON line with the keys
the driver reads."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    sys.path.insert(0, ROOT)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3", "--workload", "cpr_p1_8192"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    import bench
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == bench.usable_cpus()
    assert d["cpu_baseline"]["cpu"]["usable_cpus"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("cpr_p1_8192")


def test_workload_table_is_well_formed():
    sys.path.insert(0, ROOT)
    import bench
    for name in bench.WORKLOADS:
        method, k, nx, ny, cfl, weak, case = bench.workload(name)
        assert method in ("cpr", "dg", "ndg", "sd", "fv") and case in ("vortex", "shock")
        assert (1 <= k <= 4) if method != "fv" else (k in (1, 2))
        assert nx >= 2 and ny >= 2 and cfl > 0

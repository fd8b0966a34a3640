"""Key metrics and warp-stall breakdown of every launch in an ncu report.

    python tools/ncu_summary.py REPORT.ncu-rep [...]

Profiling aid only (not part of the product path).
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "ms"),
    ("dram__bytes_read.sum", "DRAM rd"),
    ("dram__bytes_write.sum", "DRAM wr"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed", "smem wf %"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp inst"),
]


def main():
    for rep in sys.argv[1:]:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        hdr, units, data = rows[0], rows[1], rows[2:]
        col = {h: i for i, h in enumerate(hdr)}
        print(f"== {rep}")
        for d in data:
            print("  " + d[col["Kernel Name"]][:90])
            for k, name in KEYS:
                if k in col:
                    print(f"    {name:10s} {d[col[k]]} {units[col[k]]}")
            st = {h[len("smsp__pcsamp_warps_issue_stalled_"):]: float(d[i] or 0) for h, i in col.items()
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
            tot = sum(st.values()) or 1.0
            top = sorted(st.items(), key=lambda kv: -kv[1])[:8]
            print("    stalls   " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))


if __name__ == "__main__":
    main()

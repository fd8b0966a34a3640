"""Attribute an ncu SASS source page to CUDA source lines.

    python tools/sass_lines.py REPORT.ncu-rep KERNEL_REGEX CUBIN MANGLED_NAME [--launch N] [--top K]

ncu's CSV source page carries per-SASS-instruction metrics (instructions
executed, warp-stall samples) but no line mapping; `nvdisasm -g -c` of the
same cubin carries the line mapping (-lineinfo).  Joining the two on the
instruction offset gives instructions and stall samples per source line.
Profiling aid only (not part of the product path).
"""
from __future__ import annotations

import collections
import csv
import io
import re
import subprocess
import sys


def line_map(cubin: str, fn: str):
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True, check=True).stdout
    out, cur, inside = {}, None, False
    for ln in dis.splitlines():
        if ln.startswith(".text.") or "--------------------- .text." in ln:
            inside = fn in ln
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            if "inlined at" not in ln:
                cur = (m.group(1).rsplit("/", 1)[-1], int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            out[int(m.group(1), 16)] = cur
    return out


def main():
    rep, kre, cubin, fn = sys.argv[1:5]
    launch = int(sys.argv[sys.argv.index("--launch") + 1]) if "--launch" in sys.argv else 0
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre,
                          "--launch-skip", str(launch), "--launch-count", "1"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
    h = rows[hi]
    ia, ie, iss = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    body = [r for r in rows[hi + 1:] if len(r) > ie and r[ia].startswith("0x")]
    a0 = int(body[0][ia], 16)
    lm = line_map(cubin, fn)
    inst, samp = collections.Counter(), collections.Counter()
    for r in body:
        key = lm.get(int(r[ia], 16) - a0, ("?", 0))
        inst[key] += float(r[ie] or 0)
        samp[key] += float(r[iss] or 0)
    ti, ts = sum(inst.values()), sum(samp.values())
    print(f"instructions {ti:.4g}  stall samples {ts:.4g}")
    for key, v in sorted(inst.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{100 * v / ti:5.1f}% inst  {100 * samp[key] / ts:5.1f}% samples  {key[0]}:{key[1]}")


if __name__ == "__main__":
    main()

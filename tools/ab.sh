#!/bin/bash
# A/B timing of library variants (profiling aid): LIBS="x.so y.so" WLS="wl1 wl2" REP=2 tools/ab.sh tag
# -> gpurun_out/ab_<tag>.jsonl, one bench line per (rep, workload, library), libraries interleaved
cd $GRAFT_REPO_ROOT
out=gpurun_out/ab_$1.jsonl; rm -f $out
for rep in $(seq ${REP:-2}); do
  for wl in $WLS; do
    for lib in $LIBS; do
      l=$(HOM2D_LIB=$PWD/paper_1709_01619_b200/$lib timeout 300 python bench.py --workload $wl --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline --no-tte --no-weak 2>/dev/null | tail -1)
      echo "{\"lib\": \"$lib\", \"rep\": $rep, \"line\": $l}" >> $out
    done
  done
done
python - $out <<'PY'
import json, sys
for ln in open(sys.argv[1]):
    d = json.loads(ln); b = d["line"]
    print(f'{d["rep"]} {b["config"]["workload"]:>18} {d["lib"]:>24} {b["value"]/1e9:7.2f} G  frac {b["roofline"]["frac"]:.3f}')
PY

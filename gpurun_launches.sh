#!/bin/bash
# per-launch durations of one bench step (profiling aid): WL=... ./gpurun_launches.sh tag
cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-20} -c ${CNT:-12} --csv --log-file gpurun_out/launches_$1.csv python bench.py --workload ${WL:-fv2_16384} --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-tte --no-weak > gpurun_out/launches_$1.log 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/launches_$1.csv")) if len(r)>10]
h=rows[0]
ki=h.index("Kernel Name"); vi=h.index("Metric Value")
for r in rows[1:]:
    print(r[ki][:70], r[vi])
PY

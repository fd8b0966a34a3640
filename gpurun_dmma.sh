#!/bin/bash
cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o /tmp/dmma_bench tools/dmma_bench.cu
/tmp/dmma_bench > gpurun_out/dmma_bench.txt 2>&1
cat gpurun_out/dmma_bench.txt
timeout 600 ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --csv /tmp/dmma_bench > gpurun_out/dmma_ncu.csv 2>&1
python3 - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/dmma_ncu.csv")) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); mi=h.index("Metric Name"); vi=h.index("Metric Value")
for r in rows[1:]: print(r[ki][:40], r[mi], r[vi])
PY

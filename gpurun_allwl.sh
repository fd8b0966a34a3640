#!/bin/bash
# every bench workload once (profiling aid): -> gpurun_out/bench_workloads.jsonl
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/bench_workloads.jsonl
for wl in $(python -c "import bench; print(' '.join(bench.WORKLOADS))"); do
  timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-tte --no-weak 2>/dev/null | tail -1 >> gpurun_out/bench_workloads.jsonl
done
wc -l gpurun_out/bench_workloads.jsonl

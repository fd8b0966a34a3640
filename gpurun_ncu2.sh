#!/bin/bash
# ncu --set full of one stage-2 launch per workload (profiling aid): ./gpurun_ncu2.sh "wl:kernelregex ..."
cd $GRAFT_REPO_ROOT
for v in $1; do
  wl=${v%%:*}; kre=${v##*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$kre --launch-skip ${LSKIP:-4} -c 1 -o gpurun_out/ncu_$wl -f python bench.py --workload $wl --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-tte --no-weak > gpurun_out/ncu_$wl.log 2>&1
  echo "$wl rc=$?"
done

#!/bin/bash
# ncu evidence for one build (run under gpurun): launch list of one bench step + one --set full capture per kernel
R=${1:-r2}
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${R}_launches_c3.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-latency > gpurun_out/${R}_bench_under_ncu.log 2>&1
for k in gicp_nn gicp_step gicp_init render_kernel cost_kernel; do
  skip=8; case $k in gicp_init|render_kernel|cost_kernel) skip=0;; esac
  ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -o gpurun_out/${R}_$k \
      python tools/profile_step.py --workload c3 --steps 0 > /dev/null 2>&1
done
ls -la gpurun_out/${R}_*

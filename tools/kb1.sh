#!/bin/bash
# quick C1 (small-N latency) timing: tools/kb1.sh [extra nvcc flags]
PX_NVCC_EXTRA="$*" python -c "import __graft_entry__ as g; g.build(force=True)" || exit 1
PX_NVCC_EXTRA="$*" python bench.py --workload c1 --steps 20 --warmup 3 --no-cpu --no-latency 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
k=d['roofline']['kernels']
print('[$*] c1 ms/step %.3f | nn %.3f step %.3f init %.3f | estimate_poses %.2f' % (d['ms_per_step'], k['gicp_nn_kernel']['ms_per_step'], k['gicp_step_kernel']['ms_per_step'], k['gicp_init_kernel']['ms_per_step'], d['e2e']['estimate_poses_ms']))"

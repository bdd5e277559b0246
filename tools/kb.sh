#!/bin/bash
# quick per-kernel timing of the C3 step: tools/kb.sh [extra nvcc flags]
PX_NVCC_EXTRA="$*" python -c "import __graft_entry__ as g; g.build(force=True)" || exit 1
PX_NVCC_EXTRA="$*" python bench.py --steps 3 --warmup 3 --no-cpu --no-latency 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
k=d['roofline']['kernels']
print('[$*] ms/step %.2f stage %s | nn %.2f step %.2f halve %.2f init %.2f render %.2f cost %.2f' % (d['ms_per_step'], {a:round(b,1) for a,b in d['stage_ms'].items()}, k['gicp_nn_kernel']['ms_per_step'], k['gicp_step_kernel']['ms_per_step'], k.get('gicp_halve_kernel', {}).get('ms_per_step', 0.0), k['gicp_init_kernel']['ms_per_step'], k['render_kernel']['ms_per_step'], k['cost_kernel']['ms_per_step']))"

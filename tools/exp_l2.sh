#!/bin/bash
# experiment: L2-blocked chunks (small per-chunk scratch) with / without streaming cache hints
for hints in "" "-DPX_NO_STREAM_HINTS"; do
  PX_NVCC_EXTRA="$hints" python -c "import __graft_entry__ as g; g.build(force=True)"
  for mb in 8192 1024 512 256 128; do
    PX_NVCC_EXTRA="$hints" PX_SCRATCH_MB=$mb python bench.py --steps 3 --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
k=d['roofline']['kernels']
print('hints=[$hints] mb=$mb ms/step %.2f stage %s  nn %.2f step %.2f halve %.2f init %.2f' % (d['ms_per_step'], {a:round(b,1) for a,b in d['stage_ms'].items()}, k['gicp_nn_kernel']['ms_per_step'], k['gicp_step_kernel']['ms_per_step'], k.get('gicp_halve_kernel', {}).get('ms_per_step', 0.0), k['gicp_init_kernel']['ms_per_step']))"
  done
done

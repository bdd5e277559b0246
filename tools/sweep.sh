#!/bin/bash
# usage: tools/sweep.sh "<nvcc extra flags>" ... ; rebuilds libpx.so per variant and prints stage times
for v in "$@"; do
  PX_NVCC_EXTRA="$v" python -c "import __graft_entry__ as g; g.build(force=True)" > /dev/null 2>&1
  echo "== $v: $(python tools/profile_step.py --workload ${WL:-c3} --steps 3 2>&1 | tail -1)"
done

#!/bin/bash
# usage: tools/sweep.sh "<nvcc extra flags>" ... ; rebuilds libpx.so per variant and prints stage times
for v in "$@"; do
  if PX_NVCC_EXTRA="$v" python -c "import __graft_entry__ as g; g.build(force=True)" > /tmp/sweep_build.log 2>&1; then
    echo "== $v: $(python tools/profile_step.py --workload ${WL:-c3} --steps 3 2>&1 | tail -1)"
  else
    echo "== $v: BUILD FAILED: $(grep -m1 error /tmp/sweep_build.log)"
  fi
done

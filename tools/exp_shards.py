"""experiment: one scene, candidates sharded over K device contexts / streams on ONE GPU (tails of one
stream's kernels filled by the other's)."""
import sys, time, threading
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import bench
from paper_2008_00326_b200.batch import engine_pool
from paper_2008_00326_b200.search import plan_lattice, _device_search

frame, models, cfg, plan = bench.build_workload("c3", 1, 1, materialise_targets=False)
lat = plan_lattice(frame, models, cfg)
for K in (1, 2, 3, 4):
    engs = engine_pool(K)
    out = [None] * K
    def work(r):
        out[r] = _device_search(engs[r], frame, models, lat, (r, K))
    for rep in range(3):
        t0 = time.perf_counter()
        th = [threading.Thread(target=work, args=(r,)) for r in range(K)]
        [t.start() for t in th]; [t.join() for t in th]
        dt = time.perf_counter() - t0
    keys = {o: min(out[r][0][o][0] for r in range(K) if o in out[r][0]) for o in lat.active}
    print(f"K={K}: {dt*1e3:.1f} ms wall, {lat.n/dt:.0f} poses/s, keys {sorted(keys.values())[:3]}")

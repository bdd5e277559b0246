"""Where the milliseconds of one public estimate_poses call go (C1 / C3), host-timed with device syncs."""
import sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, golden_io as G
import bench
from paper_2008_00326_b200.engine import default_engine
from paper_2008_00326_b200.search import plan_lattice, _assemble

eng = default_engine()
for wl in ("c1", "c3"):
    frame, models, cfg, _ = bench.build_workload(wl, 1, 1, materialise_targets=False)
    acc = {}
    for rep in range(6):
        t = [time.perf_counter()]
        def lap(name):
            eng.sync(); t.append(time.perf_counter())
            if rep >= 2: acc.setdefault(name, []).append((t[-1] - t[-2]) * 1e3)
        plan = plan_lattice(frame, models, cfg); lap("plan_lattice (host)")
        plan.n_observed = eng.upload_frame(frame, cfg.stride); lap("upload_frame (+observed cloud on device)")
        eng._model_keys.clear(); eng.upload_models({o: models[o] for o in plan.active}); lap("upload_models")
        eng.search_upload_lattice(plan, 0, 1); lap("lattice + targets + covariances (device)")
        sc = eng.search_cfg(plan); eng.search_run(sc); lap("search_run")
        eng.search_reduce(); win = eng.search_winners(); sm = eng.stage_millis(); lap("reduce + winners download")
        winners = {o: win[o][:5] for o in plan.active if o in win}
        _assemble(plan, winners, sm, t[0], 0); lap("assemble (host)")
    print(wl, plan.n, "candidates:", {k: round(float(np.median(v)), 3) for k, v in acc.items()}, "sum", round(sum(float(np.median(v)) for v in acc.values()), 2))

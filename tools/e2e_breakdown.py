"""Where the end-to-end (host buffers in / results out) time of one step goes."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import bench
import numpy as np
from paper_2008_00326_b200.engine import Engine
wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
frame, models, cfg, plan = bench.build_workload(wl, 1, 1, materialise_targets=False)
eng = Engine(0)
idx = np.arange(plan.n)
sc = eng.search_cfg(plan)
for rep in range(3):
    t = [time.perf_counter()]
    eng._scene_key = None; eng._model_keys.clear()
    eng.upload_scene(frame, plan.cfg.stride, plan.observed, plan.obs_labels); eng.sync(); t.append(time.perf_counter())
    eng.upload_models({oid: models[oid] for oid in plan.active}); eng.sync(); t.append(time.perf_counter())
    eng.build_targets(plan); eng.sync(); t.append(time.perf_counter())
    n = eng.search_upload(plan, idx); eng.sync(); t.append(time.perf_counter())
    eng.search_run(sc); eng.sync(); t.append(time.perf_counter())
    out = eng.search_download(n); t.append(time.perf_counter())
    names = ["scene", "models", "targets", "cand_upload", "search", "download"]
    print(rep, {k: round((b - a) * 1e3, 2) for k, a, b in zip(names, t, t[1:])}, "total", round((t[-1] - t[0]) * 1e3, 2))

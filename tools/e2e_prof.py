import sys, time, cProfile, pstats
from pathlib import Path
ROOT = Path('/root/repo'); sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import bench, numpy as np
from paper_2008_00326_b200.engine import Engine
frame, models, cfg, plan = bench.build_workload("c3", 1, 1, materialise_targets=False)
eng = Engine(0); idx = np.arange(plan.n); sc = eng.search_cfg(plan)
def step():
    eng._scene_key = None; eng._model_keys.clear()
    eng.prepare_plan(frame, models, plan); n = eng.search_upload(plan, idx); eng.search_run(sc); return eng.search_download(n)
for _ in range(2): step()
pr = cProfile.Profile(); pr.enable()
for _ in range(5): step()
pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(14)

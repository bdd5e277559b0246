"""Minimal driver for ncu: build a workload, make it resident, run the fused
search `--steps` times.  No timing claims are made from runs under a profiler."""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c3s")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--scale", type=int, default=1)
a = ap.parse_args()
from paper_2008_00326_b200.engine import Engine  # noqa: E402

frame, models, cfg, plan = bench.build_workload(a.workload, 1, a.scale, materialise_targets=False)  # targets cropped on the device, as estimate_poses does
eng = Engine(0)
eng.prepare_plan(frame, models, plan)
eng.set_kernel_timing(True)
n = eng.search_upload(plan)
sc = eng.search_cfg(plan)
for _ in range(a.steps):
    eng.search_run(sc)
import time
t0 = time.perf_counter()
eng.search_run(sc)
eng.sync()
out = eng.search_download(n)
print("kernel_ms", {k: round(v[0], 2) for k, v in eng.kernel_ms().items()})
print("candidates", n, "stage_ms", out.stage_millis, "wall_ms", (time.perf_counter() - t0) * 1e3)

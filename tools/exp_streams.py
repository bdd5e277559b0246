import sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, golden_io as G
from paper_2008_00326_b200 import estimate_poses_many
d = G.load("c1_box_3dof")
frame, models, cfg = G.frame_of(d), G.models_of(d), G.config_of(d)
jobs = [(frame, models, cfg)] * 64
for k in (1, 2, 4, 8, 16):
    estimate_poses_many(jobs[:k * 2], streams=k)
    t0 = time.perf_counter(); r = estimate_poses_many(jobs, streams=k); dt = time.perf_counter() - t0
    print(f"streams {k}: {dt / 64 * 1e3:.2f} ms/scene, {r[0].proposals_evaluated * 64 / dt:.0f} poses/s")

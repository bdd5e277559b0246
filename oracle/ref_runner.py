"""TEST / BENCH INFRASTRUCTURE -- never imported by the product.

Runs the UNMODIFIED reference package (`rvpose`, installed by `make -C oracle ref` into the git-ignored
oracle/_ref/) through its own public entry point `rvpose.search.estimate_poses` (search.py:217-377), timed the way
the reference times itself (`cli._cmd_bench`, cli.py:233-239: perf_counter around the call, file I/O excluded), with
`workers = os.cpu_count()`.  Used by `bench.py --impl reference` as the CPU arm when the package is importable on the
box (it needs numba); the C port oracle/px_oracle.c is the fallback and the second, stricter baseline.
"""

from __future__ import annotations

import dataclasses
import os
import sys
import time
from pathlib import Path

import numpy as np

REF_DIR = Path(__file__).resolve().parent / "_ref"


def available() -> str | None:
    """None when rvpose can be imported from oracle/_ref, else the reason."""
    if not (REF_DIR / "rvpose" / "search.py").exists():
        return "oracle/_ref/rvpose not installed (make -C oracle ref needs /root/reference)"
    try:
        import numba  # noqa: F401
    except Exception as e:  # pragma: no cover
        return f"numba unavailable: {e}"
    return None


def load():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/px_numba_cache")  # the package dir may be read-only
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import rvpose  # noqa: F401
    from rvpose import search
    return search


def patches_3dof(cfg, cells: int, count: int):
    """`count` sub-workspaces of cells x cells grid cells, aligned with the workload's own lattice
    (proposals._inclusive_range values) and spread uniformly over it."""
    from paper_2008_00326_b200.proposals import _inclusive_range

    x0, x1, y0, y1 = cfg.workspace
    xs, ys = _inclusive_range(x0, x1, cfg.dt), _inclusive_range(y0, y1, cfg.dt)
    nx, ny = max(1, xs.size - cells + 1), max(1, ys.size - cells + 1)
    side = int(np.ceil(np.sqrt(count)))
    ix = np.unique(np.round(np.linspace(0, nx - 1, side)).astype(int))
    iy = np.unique(np.round(np.linspace(0, ny - 1, side)).astype(int))
    grid = [(i, j) for i in ix for j in iy]
    pick = np.unique(np.round(np.linspace(0, len(grid) - 1, min(count, len(grid)))).astype(int))
    out = []
    for p in pick:
        i, j = grid[int(p)]
        out.append((float(xs[i]), float(xs[min(i + cells - 1, xs.size - 1)]),
                    float(ys[j]), float(ys[min(j + cells - 1, ys.size - 1)])))
    return out


def ref_config(search, cfg, **over):
    d = cfg.to_dict()
    d["workers"] = os.cpu_count() or 1
    rc = search.SearchConfig.from_dict(d)
    return dataclasses.replace(rc, max_proposals=cfg.max_proposals, **over)


def run_sample(search, frame, models, cfg, patches=None, max_proposals=None):
    """One timed pass: estimate_poses on every patch (3-DoF) or on the reference's own uniform
    `max_proposals` subsample (6-DoF).  -> (candidates scored, seconds, stage_millis summed)."""
    n, secs = 0, 0.0
    stages = {"render": 0.0, "refine": 0.0, "rerender": 0.0, "cost": 0.0}
    runs = [ref_config(search, cfg, workspace=w) for w in patches] if patches else \
        [ref_config(search, cfg, max_proposals=max_proposals)]
    for rc in runs:
        t0 = time.perf_counter()
        res = search.estimate_poses(frame, models, rc)
        secs += time.perf_counter() - t0
        n += int(res.proposals_evaluated)
        for k in stages:
            stages[k] += float(res.stage_millis.get(k, 0.0))
    return n, secs, stages

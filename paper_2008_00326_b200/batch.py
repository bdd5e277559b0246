"""Multi-scene batching.

A small scene (BASELINE configs[0]: ~2k candidates) cannot fill a B200: its 120-odd kernel launches are
bounded by the slowest candidate of each launch, not by throughput.  Scenes are independent (the reference
processes them one CLI invocation at a time, cli.py:192-211; scene directories scenegen.py:567-589), so
several of them run CONCURRENTLY here: a pool of device contexts (px_ctx), each with its own CUDA stream,
driven by one host thread each -- the C-ABI calls release the GIL, the streams' kernels interleave on the SMs,
and loading / planning the next scene overlaps the GPU work of the current ones.  Every scene is still scored
by exactly the single-scene code path, so its results are byte-identical to a plain `estimate_poses` call.
"""

from __future__ import annotations

import os
import threading
from concurrent.futures import ThreadPoolExecutor

from .engine import Engine
from .search import estimate_poses

_pool_lock = threading.Lock()
_pools: dict = {}


def engine_pool(streams: int, device: int | None = None) -> list:
    """`streams` contexts on one device (created once per process, serially)."""
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    with _pool_lock:
        pool = _pools.setdefault(device, [])
        while len(pool) < streams:
            pool.append(Engine(device))
        return pool[:streams]


def estimate_poses_many(jobs, streams: int = 4, device: int | None = None) -> list:
    """`jobs`: iterable of (frame, models, cfg) or of callables returning such a triple (e.g. a scene-directory
    loader, so that file I/O happens inside the worker).  Returns the SearchResults in job order."""
    jobs = list(jobs)
    if not jobs:
        return []
    streams = max(1, min(int(streams), len(jobs)))
    engines = engine_pool(streams, device)
    results = [None] * len(jobs)

    def worker(slot: int):
        eng = engines[slot]
        for j in range(slot, len(jobs), streams):
            job = jobs[j]
            frame, models, cfg = job() if callable(job) else job
            results[j] = estimate_poses(frame, models, cfg, engine=eng)

    if streams == 1:
        worker(0)
        return results
    with ThreadPoolExecutor(max_workers=streams) as ex:
        for f in [ex.submit(worker, s) for s in range(streams)]:
            f.result()
    return results

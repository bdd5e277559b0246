"""Multi-GPU sharding of the flat candidate list and the one collective.

The reference parallelises over independent (object, proposal) tasks with a fork
pool and an ordered gather (pkg/src/rvpose/parallel.py:28-37); results must not
depend on the worker count (tests/test_search.py:100-106).  Here each rank (one
process per GPU) scores a shard of the candidates and the ranks agree on the
per-object winner with a single all_reduce(MIN) over packed keys

    key = (j_o + j_r) << 32 | rank_in_object

whose integer order is exactly `select_best`'s (total, index) order
(search.py:178-183).  Nothing else crosses NVLink.  Works with any
torch.distributed backend (nccl on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

import numpy as np

NO_KEY = (1 << 63) - 1  # "no candidate on this rank" (fits int64, larger than any real key)


def shard_index(plan, rank: int, world: int) -> np.ndarray:
    """Indices (into the plan's flat list) owned by `rank`.

    Grid cells (3-DoF) / rotation hypotheses (6-DoF) are dealt round-robin, so a
    GICP target and its covariances are needed on one rank only, and the
    cheap/expensive regions of the workspace are interleaved across ranks."""
    if world <= 1:
        return np.arange(plan.n)
    key = np.empty(plan.n, dtype=np.int64)
    for oid in plan.active:
        sel = np.nonzero(plan.flat_oid == oid)[0]
        key[sel] = plan.proposal_sets[oid].provenance[plan.flat_local[sel], 0]
    return np.nonzero(key % world == rank)[0]


def pack_keys(plan, index, j_o, j_r) -> np.ndarray:
    """Per active object: min over this rank's candidates of the packed key."""
    total = j_o.astype(np.int64) + j_r.astype(np.int64)
    rank_in_obj = plan.rank_in_object()[index].astype(np.int64)
    oid = plan.flat_oid[index]
    keys = np.full(len(plan.active), NO_KEY, dtype=np.int64)
    for s, o in enumerate(plan.active):
        m = oid == o
        if m.any():
            keys[s] = int(((total[m] << 32) | rank_in_obj[m]).min())
    return keys


def keys_from_device(plan, best_keys: dict) -> np.ndarray:
    """Same, from the fused device argmin (px_search_download's best_key_per_model)."""
    return np.array([min(int(best_keys.get(o, NO_KEY)), NO_KEY) for o in plan.active], dtype=np.int64)


def allreduce_min(keys: np.ndarray, device=None) -> np.ndarray:
    """all_reduce(MIN) of the packed keys; identity when not distributed."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return keys
    t = torch.from_numpy(np.ascontiguousarray(keys))
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return t.cpu().numpy()


def unpack_key(key: int):
    """-> (total cost, rank_in_object) or None."""
    key = int(key)
    if key >= NO_KEY:
        return None
    return key >> 32, key & 0xFFFFFFFF

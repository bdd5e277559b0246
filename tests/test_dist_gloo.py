"""world_size-2 gloo test of the N>1 path (CPU): candidate sharding + the
all_reduce(MIN) of packed (cost, pose-id) keys reproduce the single-process
per-object argmin (reference tests/test_search.py:100-106: results independent
of the worker count).  Per-candidate costs come from the CPU oracle here; on the
GPU box the same host logic wraps the device engine (bench.py)."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, out_dir):
    import dataclasses

    import torch.distributed as dist

    import golden_io as G
    from oracle import oracle as O
    from paper_2008_00326_b200 import dist as pxd
    from paper_2008_00326_b200.search import plan_search

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = G.load(name)
    frame, models = G.frame_of(d), G.models_of(d)
    cfg = dataclasses.replace(G.config_of(d), max_proposals=None, dt=0.16, refine=False)
    plan = plan_search(frame, models, cfg)
    idx = pxd.shard_index(plan, rank, world)
    out = O.run_plan(frame, models, plan, n_threads=2, index=idx)
    keys = pxd.allreduce_min(pxd.pack_keys(plan, idx, out.j_o, out.j_r))
    np.save(Path(out_dir) / f"keys_{rank}.npy", keys)
    np.save(Path(out_dir) / f"idx_{rank}.npy", idx)
    dist.destroy_process_group()


def test_two_rank_argmin_equals_single_process(tmp_path):
    import dataclasses

    import golden_io as G
    from oracle import oracle as O
    from paper_2008_00326_b200 import dist as pxd
    from paper_2008_00326_b200.search import assemble_result, plan_search

    name, world = "c3_clutter_3dof", 2
    mp.spawn(_worker, args=(world, _free_port(), name, str(tmp_path)), nprocs=world, join=True)
    d = G.load(name)
    frame, models = G.frame_of(d), G.models_of(d)
    cfg = dataclasses.replace(G.config_of(d), max_proposals=None, dt=0.16, refine=False)
    plan = plan_search(frame, models, cfg)
    idx = [np.load(tmp_path / f"idx_{r}.npy") for r in range(world)]
    # shards partition the candidate list and keep grid cells together
    assert np.array_equal(np.sort(np.concatenate(idx)), np.arange(plan.n))
    for oid in plan.active:
        cells = [set(plan.proposal_sets[oid].provenance[plan.flat_local[i[plan.flat_oid[i] == oid]], 0]) for i in idx]
        assert not (cells[0] & cells[1])
    k0, k1 = (np.load(tmp_path / f"keys_{r}.npy") for r in range(world))
    assert np.array_equal(k0, k1)  # every rank knows the winners
    single = O.run_plan(frame, models, plan, n_threads=2)
    res = assemble_result(plan, single, 0.0)
    for s, oid in enumerate(plan.active):
        e = res.estimate_for(oid)
        assert pxd.unpack_key(k0[s]) == (e.cost.total, e.proposal_index)
    assert np.array_equal(pxd.pack_keys(plan, np.arange(plan.n), single.j_o, single.j_r), k0)


def test_shard_index_world1_and_keys():
    import golden_io as G
    from paper_2008_00326_b200 import dist as pxd

    d, frame, models, cfg, plan = G.scene("c4_mixed_6dof")
    assert np.array_equal(pxd.shard_index(plan, 0, 1), np.arange(plan.n))
    parts = [pxd.shard_index(plan, r, 4) for r in range(4)]
    assert np.array_equal(np.sort(np.concatenate(parts)), np.arange(plan.n))
    assert pxd.unpack_key(pxd.NO_KEY) is None and pxd.unpack_key((7 << 32) | 5) == (7, 5)
    assert np.array_equal(pxd.keys_from_device(plan, {}), np.full(len(plan.active), pxd.NO_KEY))


def _worker_api(rank, world, port, name, out_dir):
    import dataclasses

    import torch.distributed as dist

    import golden_io as G
    from oracle import oracle as O
    from paper_2008_00326_b200.search import estimate_poses_distributed, result_to_json

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = G.load(name)
    frame, models = G.frame_of(d), G.models_of(d)
    cfg = dataclasses.replace(G.config_of(d), max_proposals=600)

    def runner(frame, models, plan, index):  # the CPU checker stands in for the device engine
        return O.run_plan(frame, models, plan, n_threads=2, index=index)

    res = estimate_poses_distributed(frame, models, cfg, runner=runner)
    (Path(out_dir) / f"result_{rank}.json").write_text(result_to_json(res))
    dist.destroy_process_group()


def test_estimate_poses_distributed_equals_single_process(tmp_path):
    """The public multi-rank entry (refine on, winners' refined poses travelling through the
    second all_reduce): every rank returns the single-process result JSON byte for byte."""
    import dataclasses

    import golden_io as G
    from oracle import oracle as O
    from paper_2008_00326_b200.search import assemble_result, plan_search, result_to_json

    name, world = "c1_box_3dof", 2
    mp.spawn(_worker_api, args=(world, _free_port(), name, str(tmp_path)), nprocs=world, join=True)
    d = G.load(name)
    frame, models = G.frame_of(d), G.models_of(d)
    cfg = dataclasses.replace(G.config_of(d), max_proposals=600)
    plan = plan_search(frame, models, cfg)
    single = result_to_json(assemble_result(plan, O.run_plan(frame, models, plan, n_threads=2), 0.0))
    for r in range(world):
        assert (tmp_path / f"result_{r}.json").read_text() == single

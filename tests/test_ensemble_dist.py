"""Multi-process (gloo, world size 2, CPU) coverage of the ensemble path:
deterministic sharding, every cell solved exactly once, results gathered on
every rank.  The per-cell solver is a CPU stub here; on GPU boxes the same
driver runs ``ensemble.permeability_job`` per rank."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_15554_b200 import ensemble
from paper_2312_15554_b200.grid import UnitCellGrid, make_model_geometry


def _jobs():
    radii = [0.1, 0.15, 0.2, 0.25, 0.3, 0.35, 0.4]
    jobs = []
    for i, r in enumerate(radii):
        ind = make_model_geometry(UnitCellGrid((8 + 4 * (i % 3),) * 3), radius=r)
        jobs.append(ensemble.CellJob(key=("cell", i), indicator=ind,
                                     cost=ensemble.default_cost(ind, 100 + 10 * i)))
    return jobs


def _stub(job):
    ind = job.indicator
    return {"porosity": 1.0 - float(ind.values.mean()), "rank": dist.get_rank() if dist.is_initialized() else 0,
            "n": int(ind.values.size)}


def test_shard_is_a_balanced_partition():
    jobs = _jobs()
    for world in (1, 2, 3, 4, 8):
        parts = ensemble.shard(jobs, world)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(len(jobs)))
        loads = [sum(jobs[i].cost for i in p) for p in parts]
        assert max(loads) - min(loads) <= max(j.cost for j in jobs)
        assert parts == ensemble.shard(jobs, world)  # deterministic


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = ensemble.run_ensemble(_jobs(), _stub)
        out_q.put((rank, {k: v for k, v in res.items()}))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_run_ensemble_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    jobs = _jobs()
    parts = ensemble.shard(jobs, 2)
    for rank in (0, 1):
        res = results[rank]
        assert set(res) == {j.key for j in jobs}
        for i, j in enumerate(jobs):
            owner = 0 if i in parts[0] else 1
            assert res[j.key]["rank"] == owner
            assert res[j.key]["porosity"] == pytest.approx(1.0 - float(j.indicator.values.mean()))
    assert results[0] == results[1]


def test_run_ensemble_single_process_runs_everything():
    res = ensemble.run_ensemble(_jobs(), _stub)
    assert len(res) == len(_jobs())
    assert all(np.isfinite(v["porosity"]) for v in res.values())
